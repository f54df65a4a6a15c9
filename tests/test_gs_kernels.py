"""Every Gauss-Seidel sweep kernel against the oracle.

The setup-time rule (amg_cycle.cu: tune_level_sweep) picks, per AMG level, one
of the dependency-scheduled sweep kernels (level-synchronous step programs as
one group or a pipeline of groups, with one or several lockstep warps and a
dependency class of 2, 4 or 8 per node; thread-block cluster; warp per row);
all of them keep the natural-order semantics of sym_gauss_seidel
(amg.cpp:25-43).  Each is forced here (MPREC_GS_MODE, MPREC_GS_LS_K,
MPREC_GS_LS_NW, MPREC_GS_LS_ND) on config 2, and the preconditioner apply /
solve are checked against the oracle.
"""

import numpy as np
import pytest

from paper_1912_04385_b200 import gen
from tests.systems import random_vec

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def cfg2():
    return gen.generate(2)


LS_MODES = {
    # groups, warps per group, dependency class (0: from the level)
    "ls": ("16", "1", "0"),
    "ls-k1": ("1", "1", "0"),          # one group: no boundary, far dependencies through the own importer
    "ls-k1-nw4": ("1", "4", "0"),      # lockstep warps, named barrier per step
    "ls-k37-nw2": ("37", "2", "0"),
    "ls-nd4": ("8", "1", "4"),         # rows wider than 4 dependencies become partial-node trees
    "ls-nd8": ("4", "2", "8"),
    "ls-k1-far": ("1", "2", "0"),      # + a 512-slot ring: most dependencies return through the own importer
}


@pytest.mark.parametrize("mode", ["warp", "cluster", *LS_MODES, ""])
@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg"])
def test_forced_sweep_kernel(gpu, orc, cfg2, mode, method, monkeypatch):
    if mode in LS_MODES:
        k, nw, nd = LS_MODES[mode]
        monkeypatch.setenv("MPREC_GS_LS_K", k)
        monkeypatch.setenv("MPREC_GS_LS_NW", nw)
        monkeypatch.setenv("MPREC_GS_LS_ND", nd)
        if mode == "ls-k1-far":
            monkeypatch.setenv("MPREC_GS_LS_WCAP", "512")
        mode = "ls"
    monkeypatch.setenv("MPREC_GS_MODE", mode)
    a, b, _ = cfg2
    sg = gpu.system(a).setup(method, b)
    so = orc.system(a).setup(method, b)
    r = random_vec(a.dim, 11)
    assert rel(sg.apply(r), so.apply(r)) < 1e-10
    for st in range(so.n_stages() - 1):
        assert rel(sg.apply_stage(st, r), so.apply_stage(st, r)) < 1e-10, f"stage {st}"
    rg, ro = sg.solve(), so.solve()
    assert abs(rg.iterations - ro.iterations) <= 1
    assert rg.converged == ro.converged
    assert rel(rg.x, ro.x) < 1e-6


@pytest.mark.parametrize("groups", ["32", "148", "0"])
@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg"])
def test_ilu_level_sync_solve(gpu, orc, cfg2, method, groups, monkeypatch):
    """Block ILU(0) solves against the oracle: the level-synchronous solve streams
    (ilu_ls.cu, default; 32 and 148 groups) and the warp-per-block-row kernel
    (ilu_solve.cu, MPREC_ILU_LS=0)."""
    monkeypatch.setenv("MPREC_ILU_LS", groups)
    a, b, _ = cfg2
    sg = gpu.system(a).setup(method, b)
    so = orc.system(a).setup(method, b)
    r = random_vec(a.dim, 5)
    assert rel(sg.apply(r), so.apply(r)) < 1e-10
    rg, ro = sg.solve(), so.solve()
    assert abs(rg.iterations - ro.iterations) <= 1
    assert rel(rg.x, ro.x) < 1e-6
