"""GPU (sm_100a library) vs CPU oracle parity on the solve path.

Bars (BASELINE.json north_star): C/F splittings, sparsity patterns and the
exact setup values (scaled system, extracted sub-systems, ILU(0) factors,
interpolation and Galerkin operators) bitwise; preconditioner applications
and solutions within 1e-10 relative; GMRES iteration counts within +-1; the
final true residual at or below the same tolerance.
"""
import numpy as np
import pytest

from paper_1912_04385_b200 import gen
from tests.systems import SMALL_SPECS, random_vec, small_system

pytestmark = pytest.mark.gpu

METHODS = ["cpr-amg", "cptr3-amg"]
APPLY_TOL = 1e-10


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _pair(gpu, orc, a, b, method, **amg):
    return gpu.system(a).setup(method, b, **amg), orc.system(a).setup(method, b, **amg)


def _check_hierarchy(hg, ho):
    assert hg.n_levels == ho.n_levels
    for l in range(ho.n_levels):
        assert hg.level_info(l) == ho.level_info(l), f"level {l} sizes"
        for which in ([0] if l == 0 else [0, 1, 2]):
            g_rp, g_ci, g_v = hg.level_csr(l, which)
            o_rp, o_ci, o_v = ho.level_csr(l, which)
            assert np.array_equal(g_rp, o_rp) and np.array_equal(g_ci, o_ci), f"level {l} pattern {which}"
            assert np.array_equal(g_v, o_v), f"level {l} values {which} (max diff {np.abs(g_v - o_v).max()})"
        if l + 1 < ho.n_levels:
            assert np.array_equal(hg.cf(l), ho.cf(l)), f"C/F splitting of level {l}"


@pytest.mark.parametrize("name", list(SMALL_SPECS))
@pytest.mark.parametrize("method", METHODS)
def test_setup_bitwise(gpu, orc, name, method):
    a, b, _ = small_system(name)
    sg, so = _pair(gpu, orc, a, b, method, max_coarse_size=40)
    ag, bg = sg.scaled()
    ao, bo = so.scaled()
    assert np.array_equal(ag, ao), "scaled matrix"
    assert np.array_equal(bg, bo), "scaled rhs"
    assert np.array_equal(sg.ilu_values(), so.ilu_values()), "ILU(0) factors"
    assert sg.n_stages() == so.n_stages()
    for st in range(so.n_stages() - 1):
        _check_hierarchy(sg.stage_amg(st), so.stage_amg(st))


@pytest.mark.parametrize("name", list(SMALL_SPECS))
@pytest.mark.parametrize("method", METHODS)
def test_apply_parity(gpu, orc, name, method):
    a, b, _ = small_system(name)
    sg, so = _pair(gpu, orc, a, b, method, max_coarse_size=40)
    r = random_vec(a.dim, 5)
    assert rel(sg.apply(r), so.apply(r)) < APPLY_TOL
    for st in range(so.n_stages()):
        assert rel(sg.apply_stage(st, r), so.apply_stage(st, r)) < APPLY_TOL, f"stage {st}"
    assert rel(sg.spmv(r, 0), so.spmv(r, 0)) < 1e-13
    assert rel(sg.spmv(r, 1), so.spmv(r, 1)) < 1e-13


@pytest.mark.parametrize("name", list(SMALL_SPECS))
@pytest.mark.parametrize("method", METHODS)
def test_solve_parity(gpu, orc, name, method):
    a, b, xs = small_system(name)
    sg, so = _pair(gpu, orc, a, b, method, max_coarse_size=40)
    rg, ro = sg.solve(), so.solve()
    assert rg.converged == ro.converged
    assert abs(rg.iterations - ro.iterations) <= 1, (rg.iterations, ro.iterations)
    if ro.converged:
        assert rg.final_true_residual <= 1e-8
    n = min(len(rg.residual_history), len(ro.residual_history))
    np.testing.assert_allclose(rg.residual_history[:n], ro.residual_history[:n], rtol=1e-6, atol=1e-14)
    assert rel(rg.x, ro.x) < 1e-6


@pytest.mark.parametrize("method", ["cpr-direct", "cptr-direct", "cptr3-direct"])
def test_direct_methods_parity(gpu, orc, method):
    a, b, xs = small_system("g12x10_nb4_band")
    sg, so = _pair(gpu, orc, a, b, method)
    ag, bg = sg.scaled()
    ao, bo = so.scaled()
    assert np.array_equal(ag, ao) and np.array_equal(bg, bo)
    assert np.array_equal(sg.ilu_values(), so.ilu_values())
    r = random_vec(a.dim, 5)
    assert rel(sg.apply(r), so.apply(r)) < APPLY_TOL
    rg, ro = sg.solve(), so.solve()
    assert abs(rg.iterations - ro.iterations) <= 1 and rg.converged == ro.converged
    assert rel(rg.x, ro.x) < 1e-6


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_baseline_configs_small(gpu, orc, cid):
    """BASELINE.json configs 1-3 at full size: setup bitwise, iterations +-1."""
    a, b, xs = gen.generate(cid)
    for method in gen.CONFIG_METHODS[cid]:
        sg, so = _pair(gpu, orc, a, b, method)
        ag, bg = sg.scaled()
        ao, bo = so.scaled()
        assert np.array_equal(ag, ao) and np.array_equal(bg, bo)
        for st in range(so.n_stages() - 1):
            hg, ho = sg.stage_amg(st), so.stage_amg(st)
            assert hg.n_levels == ho.n_levels
            for l in range(ho.n_levels - 1):
                assert np.array_equal(hg.cf(l), ho.cf(l)), f"stage {st} level {l} C/F"
        assert np.array_equal(sg.ilu_values(), so.ilu_values())
        rg, ro = sg.solve(), so.solve()
        assert abs(rg.iterations - ro.iterations) <= 1, (method, rg.iterations, ro.iterations)
        assert rg.converged == ro.converged
        assert rel(rg.x, ro.x) < 1e-6
