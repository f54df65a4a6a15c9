"""Per-config table (BASELINE configs 1-4): GPU vs CPU oracle, both methods where
BASELINE names two, plus the per-kernel-class time split of the GPU solve and
the per-stage split of one preconditioner application (CUDA events per launch;
BASELINE config 3 asks for the per-stage kernel time split).  Writes JSON to stdout.

    python scripts/config_table.py [cids] [--no-oracle]
"""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

KCLASS = ["spmv", "spmv_col", "ilu_fwd", "ilu_bwd", "gs", "csr", "coarse", "mgs", "blas1"]
args = [x for x in sys.argv[1:] if not x.startswith("--")]
cids = [int(x) for x in args[0].split(",")] if args else [1, 2, 3, 4]
with_oracle = "--no-oracle" not in sys.argv
g = gpu()
orc = None
if with_oracle:
    import oracle
    orc = oracle.api()
rows = []
for cid in cids:
    a, b, xs = gen.generate(cid)
    for method in gen.CONFIG_METHODS[cid]:
        row = {"config": cid, "method": method, "cells": a.n_cells, "nb": a.nb}
        s = g.system(a)
        t0 = time.perf_counter()
        s.setup(method, b)
        row["gpu_setup_s"] = time.perf_counter() - t0
        s.solve(1e-8, 500)  # warm
        g.call("reset_stats", s.h)
        g.call("profile", s.h, 1)
        t0 = time.perf_counter()
        r = s.solve(1e-8, 500)
        row["gpu_solve_s"] = time.perf_counter() - t0
        g.call("profile", s.h, 0)
        split = {}
        for k, name in enumerate(KCLASS):
            tt, n, by = C.c_double(), C.c_int64(), C.c_double()
            g.call("kernel_stats", s.h, k, C.byref(tt), C.byref(n), C.byref(by))
            if n.value:
                split[name] = {"ms": round(tt.value, 3), "launches": n.value,
                               "GBps": round(by.value / max(tt.value, 1e-9) / 1e6, 1)}
        # per-stage device time of one preconditioner application (Alg. 1/2 stages:
        # temperature AMG / pressure AMG / ILU(0) for cptr3-amg): kernel time of each
        # stage applied alone to a fixed vector, mean of 10
        import numpy as np
        rv = np.random.default_rng(1).standard_normal(a.dim)
        stage_ms = []
        for st in range(s.n_stages()):
            s.apply_stage(st, rv)  # warm
            g.call("reset_stats", s.h)
            g.call("profile", s.h, 1)
            for _ in range(10):
                s.apply_stage(st, rv)
            g.call("profile", s.h, 0)
            tot = 0.0
            for k in range(len(KCLASS)):
                tt, n, by = C.c_double(), C.c_int64(), C.c_double()
                g.call("kernel_stats", s.h, k, C.byref(tt), C.byref(n), C.byref(by))
                tot += tt.value
            stage_ms.append(round(tot / 10, 4))
        row["gpu_stage_ms"] = stage_ms
        row.update(gpu_iterations=list(r.attempt_iterations), gpu_converged=r.converged,
                   gpu_true_residual=r.final_true_residual, gpu_split=split,
                   gpu_x_err=float(((r.x - xs) ** 2).sum() ** 0.5 / (xs ** 2).sum() ** 0.5))
        if orc is not None:
            so = orc.system(a)
            t0 = time.perf_counter()
            so.setup(method, b)
            row["cpu_setup_s"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            ro = so.solve(1e-8, 500)
            row["cpu_solve_s"] = time.perf_counter() - t0
            row.update(cpu_iterations=list(ro.attempt_iterations), cpu_converged=ro.converged,
                       cpu_true_residual=ro.final_true_residual)
        print(json.dumps(row), flush=True)
        rows.append(row)
