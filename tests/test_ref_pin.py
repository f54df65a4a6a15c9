"""Pins the CPU oracle to the reference's own execution.

oracle/_ref/libmprec_ref.so is the reference's unmodified sources
(/root/reference/proj/src: scaling, stages, amg, ilu0, gmres, harness,
condense, ...) compiled against the Eigen-subset shim (oracle/eigen_shim,
one fixed product / LU / dot convention) behind the same C ABI as the oracle.
These tests assert that the oracle restatement reproduces the reference's
control flow BITWISE on every value the GPU parity tests compare against the
oracle: the scaled system, the ILU(0) factors, every AMG level (C/F
splitting, P, R, A_l), the preconditioner applications, the GMRES residual
history, the iterate x and the true residual, the attempt count of
solve_system, condensation and the error classes with their payloads.
"""
import numpy as np
import pytest

from paper_1912_04385_b200 import gen
from paper_1912_04385_b200.api import DimensionError, SingularBlockError
from tests.systems import RETRY_SPECS, SMALL_SPECS, random_vec, retry_system, small_system

METHODS = ["cpr-amg", "cptr3-amg"]


def _assert_hierarchy_equal(hr, ho):
    assert hr.n_levels == ho.n_levels
    for l in range(ho.n_levels):
        assert hr.level_info(l) == ho.level_info(l)
        for which in ([0] if l == 0 else [0, 1, 2]):
            for x, y in zip(hr.level_csr(l, which), ho.level_csr(l, which)):
                assert np.array_equal(x, y), f"level {l} operator {which}"
        if l + 1 < ho.n_levels:
            assert np.array_equal(hr.cf(l), ho.cf(l)), f"C/F of level {l}"


def _assert_setup_equal(sr, so):
    ar, br = sr.scaled()
    ao, bo = so.scaled()
    assert np.array_equal(ar, ao), "scaled matrix"
    assert np.array_equal(br, bo), "scaled rhs"
    assert np.array_equal(sr.ilu_values(), so.ilu_values()), "ILU(0) factors"
    assert sr.n_stages() == so.n_stages()
    for st in range(so.n_stages() - 1):
        try:
            ho = so.stage_amg(st)
        except Exception:  # -direct stages carry no hierarchy
            continue
        _assert_hierarchy_equal(sr.stage_amg(st), ho)


def _assert_solve_equal(rr, ro):
    assert rr.iterations == ro.iterations
    assert rr.converged == ro.converged and rr.breakdown == ro.breakdown
    assert rr.attempts == ro.attempts and rr.attempt_iterations == ro.attempt_iterations
    assert np.array_equal(rr.residual_history, ro.residual_history)
    assert np.array_equal(rr.x, ro.x)
    assert rr.final_true_residual == ro.final_true_residual
    assert rr.attempt_true_residual == ro.attempt_true_residual and rr.attempt_tol == ro.attempt_tol


@pytest.mark.parametrize("name", list(SMALL_SPECS))
@pytest.mark.parametrize("method", METHODS + ["cpr-direct", "cptr-direct", "cptr3-direct", "ilu0"])
def test_small_systems_bitwise(ref, orc, name, method):
    a, b, _ = small_system(name)
    sr = ref.system(a).setup(method, b, max_coarse_size=40)
    so = orc.system(a).setup(method, b, max_coarse_size=40)
    _assert_setup_equal(sr, so)
    r = random_vec(a.dim, 3)
    assert np.array_equal(sr.apply(r), so.apply(r))
    for st in range(so.n_stages()):
        assert np.array_equal(sr.apply_stage(st, r), so.apply_stage(st, r)), f"stage {st}"
    assert np.array_equal(sr.spmv(r, 0), so.spmv(r, 0))
    assert np.array_equal(sr.spmv(r, 1), so.spmv(r, 1))
    _assert_solve_equal(sr.solve(), so.solve())


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_baseline_configs_bitwise(ref, orc, cid):
    """BASELINE configs 1-3 at full size, every method the config names."""
    a, b, _ = gen.generate(cid)
    for method in gen.CONFIG_METHODS[cid]:
        sr = ref.system(a).setup(method, b)
        so = orc.system(a).setup(method, b)
        _assert_setup_equal(sr, so)
        _assert_solve_equal(sr.solve(), so.solve())


def test_solve_system_entry_point(ref, orc):
    """ref_solve_system is the reference's own solve_system (harness.cpp:190-219),
    attempt loop included."""
    import ctypes as C

    from paper_1912_04385_b200.api import _Result, parse_method
    a, b, _ = small_system("g20x20_nb4_hiPe")
    x = np.zeros(a.dim)
    res = _Result()
    ref.call("solve_system", C.byref(a._c), b.ctypes.data, parse_method("cptr3-amg"), 1e-8, 500, x.ctypes.data,
             C.byref(res))
    ro = orc.system(a).setup("cptr3-amg", b).solve()
    assert res.iterations == ro.iterations and bool(res.converged) == ro.converged
    assert res.final_true_residual == ro.final_true_residual
    assert np.array_equal(x, ro.x)


@pytest.mark.parametrize("name", list(RETRY_SPECS))
def test_retry_loop_bitwise(ref, orc, name):
    """Systems whose scaled residual reaches tol while the true residual does
    not: the reference tightens the tolerance twice (harness.cpp:209-217)."""
    a, b, _, method = retry_system(name)
    rr = ref.system(a).setup(method, b, max_coarse_size=40).solve()
    ro = orc.system(a).setup(method, b, max_coarse_size=40).solve()
    assert ro.attempts == 3 and not ro.converged
    _assert_solve_equal(rr, ro)


def test_singular_block_error_parity(ref, orc):
    a, b, _ = small_system("g8x6_nb3")
    vals = a.values.reshape(-1, 3, 3).copy()
    d = a.row_ptr[5] + np.searchsorted(a.col_idx[a.row_ptr[5]:a.row_ptr[6]], 5)
    vals[d, :, 0] = 0.0  # D_hh of cell 5 singular: its s column is zero
    from paper_1912_04385_b200.api import BlockMatrix
    bad = BlockMatrix(a.n_cells, 3, a.row_ptr, a.col_idx, vals.reshape(-1))
    for method in ("cpr-amg", "cptr3-amg"):
        errs = []
        for api in (ref, orc):
            with pytest.raises(SingularBlockError) as e:
                api.system(bad).setup(method, b)
            errs.append((e.value.cell_id, str(e.value)))
        assert errs[0] == errs[1]
        assert errs[0][0] == 5


def test_rhs_length_error_parity(ref, orc):
    a, b, _ = small_system("g8x6_nb3")
    for api in (ref, orc):
        with pytest.raises(DimensionError):
            api.system(a).setup("cpr-amg", b[:-1])


@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg", "cptr-direct"])
@pytest.mark.parametrize("diag_mode", ["block", "scalar"])
@pytest.mark.parametrize("second", [False, True])
def test_scaling_options_bitwise(ref, orc, method, diag_mode, second):
    """ScalingOptions{diag_mode, second_scaling_from_original} (scaling.hpp:22-30)."""
    a, b, _ = small_system("g16x16_nb8_band")
    kw = dict(diag_mode=diag_mode, second_scaling_from_original=second, max_coarse_size=40)
    sr = ref.system(a).setup(method, b, **kw)
    so = orc.system(a).setup(method, b, **kw)
    _assert_setup_equal(sr, so)
    assert sr.scaling_record() == so.scaling_record()
    _assert_solve_equal(sr.solve(), so.solve())
