"""Static condensation throughput: GPU vs the CPU oracle.

python scripts/bench_condense.py [n_cells] [n_c] [n_s]
Times mprec_gpu_condense (host arrays in, device-resident reduced system out:
the H2D of the Jacobian is inside the timed call) and back_substitute on a
synthetic chain of mixed G/OG/OWG cells (condense.cpp:359-421 structure), and
the oracle on a bounded sample of the same generator.  Prints one JSON line.
"""
import ctypes as C
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import condense as cd  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 500_000
n_c = int(sys.argv[2]) if len(sys.argv) > 2 else 12
n_s = int(sys.argv[3]) if len(sys.argv) > 3 else 1
states = np.random.default_rng(3).integers(0, 3, n)
t = time.perf_counter()
pj = cd.make_synthetic_global_bulk(states, n_c, n_s, 7)
gen_s = time.perf_counter() - t
api = gpu()
red = api.condense(pj)  # warm-up (module load, allocations)
del red
ts = []
for _ in range(3):
    t = time.perf_counter()
    gj = pj.c_struct()
    h = C.c_void_p()
    api.call("condense", C.byref(gj), C.byref(h))
    ts.append(time.perf_counter() - t)
    api.fn["condensed_destroy"](h)
t_gpu = min(ts)
red = api.condense(pj)
d1 = np.random.default_rng(1).standard_normal(n * pj.np)
tb = []
for _ in range(3):
    t = time.perf_counter()
    red.back_substitute(d1)
    tb.append(time.perf_counter() - t)
out = {"metric": "condense_cells_per_s", "value": n / t_gpu, "unit": "cells/s", "n_cells": n, "n_c": n_c, "n_s": n_s,
       "np": pj.np, "n_secondary": pj.n_secondary_total, "input_GB": pj.bytes() / 1e9,
       "condense_s": t_gpu, "input_GBps_incl_h2d": pj.bytes() / t_gpu / 1e9, "back_substitute_s": min(tb),
       "generate_s": gen_s, "timer": "host wall clock around the synchronous C-ABI call (H2D included)"}
try:
    import oracle  # bounded CPU sample (the checker, not the product)
    orc = oracle.api()
    m = min(n, 20_000)
    ps = cd.make_synthetic_global_bulk(states[:m], n_c, n_s, 7)
    t = time.perf_counter()
    orc.condense(ps)
    tc = time.perf_counter() - t
    out["cpu_baseline"] = {"value": m / tc, "unit": "cells/s", "cores": 1, "kind": "port",
                           "sample": f"{m} cells of the same generator"}
except Exception as e:  # the oracle is optional for this script
    out["cpu_baseline"] = {"unavailable": str(e)}
print(json.dumps(out))
