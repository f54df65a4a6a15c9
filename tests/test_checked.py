"""Bounds-checked build (libmprec_gpu_checked.so, -DMPREC_CHECKED): the device-side
MG_DCHECKs of the sync-free and level-synchronous kernels (gs_ls.cu, ilu_ls.cu,
ilu_solve.cu) stand in for compute-sanitizer, which this GPU pool does not run.
A failed check traps the kernel; the call then fails with MPREC_CUDA.  Each
kernel variant runs in a fresh process (the library is chosen at import, the
kernel knobs are read per process) on configs 1-2 and a small reaction-band
system, and must reproduce the regular library's results."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import json, sys
import numpy as np
sys.path.insert(0, '.')
from paper_1912_04385_b200 import gen
from paper_1912_04385_b200.api import gpu
g = gpu()
out = {}
for name, spec in [('c1', 1), ('c2', 2), ('band', gen.make_spec(40, 30, 8, kappa=1.0, perm_sigma=1.5, band=True, seed=4))]:
    a, b, _ = gen.generate(spec)
    for m in ('cpr-amg', 'cptr3-amg'):
        r = g.system(a).setup(m, b, max_coarse_size=40).solve(1e-8, 60)
        out[f'{name}/{m}'] = [r.iterations, float(np.linalg.norm(r.x))]
print(json.dumps(out))
"""

VARIANTS = {
    "default": {},
    "ilu-warp": {"MPREC_ILU_LS": "0"},
    "ilu-ls32": {"MPREC_ILU_LS": "32"},
    "gs-ls-k8": {"MPREC_GS_MODE": "ls", "MPREC_GS_LS_K": "8"},
    "gs-ls-k1-nw3-nd4": {"MPREC_GS_MODE": "ls", "MPREC_GS_LS_K": "1", "MPREC_GS_LS_NW": "3", "MPREC_GS_LS_ND": "4"},
    "gs-warp": {"MPREC_GS_MODE": "warp"},
    "rs-nowindow": {"MPREC_RS_WINDOW": "0"},  # RS passes without their shared-memory windows: same results
    "rs-small-window": {"MPREC_RS_BUDGET_KB": "24"},  # 4k-point window: it moves, selections fall outside
    "rs-norecords": {"MPREC_RS_RECORDS": "0"},  # CSR walk instead of the two-hop adjacency records
}


def _run(env_extra, checked):
    env = dict(os.environ, **env_extra)
    if checked:
        env["MPREC_LIB"] = "checked"
    else:
        env.pop("MPREC_LIB", None)
    p = subprocess.run([sys.executable, "-c", CODE], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-4000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_checked_build(variant):
    if not os.path.exists(os.path.join(ROOT, "paper_1912_04385_b200", "libmprec_gpu_checked.so")):
        pytest.fail("libmprec_gpu_checked.so missing: run __graft_entry__.build()")
    ck = _run(VARIANTS[variant], True)
    rg = _run(VARIANTS[variant], False)
    assert ck == rg, (ck, rg)


def test_rs_window_does_not_change_results():
    """The windowed RS passes (amg_setup_exact.cu) are an implementation detail: without
    the windows, and with a window so small that it keeps moving and many selections
    are served from global memory, setup and solves are bit-for-bit the default's."""
    dflt = _run({}, False)
    assert _run(VARIANTS["rs-nowindow"], False) == dflt
    assert _run(VARIANTS["rs-small-window"], False) == dflt
    assert _run(VARIANTS["rs-norecords"], False) == dflt


def test_fused_residual_restriction_bitwise():
    """K15: the fused rc = R (r - A x) kernel (small levels, amg_cycle.cu) reproduces the
    two-launch path bit for bit: same iteration counts and solution norms with the
    fusion off (MPREC_FUSE_RR_MAX=0), on for every level, and at the default threshold."""
    off = _run({"MPREC_FUSE_RR_MAX": "0"}, False)
    on_all = _run({"MPREC_FUSE_RR_MAX": "2000000000"}, False)
    dflt = _run({}, False)
    assert off == on_all == dflt, (off, on_all, dflt)
