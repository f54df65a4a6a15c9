"""GPU parity of the drop-in boundary beyond the default path: ScalingOptions,
MethodSpec's -direct sub-solvers, scaling_record, the level sets of every
sequential sweep, solve_system's tolerance-tightening loop, the error classes
with their payloads, and reproducibility of setup."""
import numpy as np
import pytest

from paper_1912_04385_b200.api import (BlockMatrix, DimensionError, ScalarMatrix, SetupError, SingularBlockError,
                                       SolveResult)
from tests.ensemble import perturbed
from tests.systems import RETRY_SPECS, random_vec, retry_system, small_system

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg", "cptr-direct", "cptr3-direct"])
@pytest.mark.parametrize("diag_mode", ["block", "scalar"])
@pytest.mark.parametrize("second", [False, True])
def test_scaling_options(gpu, orc, method, diag_mode, second):
    """ScalingOptions{diag_mode, second_scaling_from_original} (scaling.hpp:22-30):
    the scaled system bitwise, the solve within the parity bars."""
    a, b, _ = small_system("g16x16_nb8_band")
    kw = dict(diag_mode=diag_mode, second_scaling_from_original=second, max_coarse_size=40)
    sg = gpu.system(a).setup(method, b, **kw)
    so = orc.system(a).setup(method, b, **kw)
    ag, bg = sg.scaled()
    ao, bo = so.scaled()
    assert np.array_equal(ag, ao) and np.array_equal(bg, bo)
    assert np.array_equal(sg.ilu_values(), so.ilu_values())
    assert sg.scaling_record() == so.scaling_record()
    rg, ro = sg.solve(), so.solve()
    assert abs(rg.iterations - ro.iterations) <= 1 and rg.converged == ro.converged
    assert rel(rg.x, ro.x) < 1e-6


def test_scaling_record_strings(gpu):
    a, b, _ = small_system("g12x10_nb4_band")
    expect = {"ilu0": "", "cpr-amg": "D_Ph*D_hh^-1", "cpr-direct": "D_Ph*D_hh^-1",
              "cptr-direct": "D_es*D_ss^-1", "cptr3-amg": "[D_Ps;D_Ts]*D_ss^-1, D_Tp*D_PP^-1",
              "cptr3-direct": "[D_Ps;D_Ts]*D_ss^-1, D_Tp*D_PP^-1"}
    for m, rec in expect.items():
        assert gpu.system(a).setup(m, b).scaling_record() == rec, m


@pytest.mark.parametrize("name", ["g16x16_nb8_band", "g30x30_nb5_loPe"])
def test_levelsets_bit_exact(gpu, orc, name):
    """north_star: the level sets of every sequential sweep the device schedules
    (GS forward/backward on every smoothed AMG level, amg.cpp:31-42; the block
    ILU(0) DAG, ilu0.cpp:16-38, 48-57) equal the reference order's level sets."""
    a, b, _ = small_system(name)
    sg = gpu.system(a).setup("cptr3-amg", b, max_coarse_size=40)
    so = orc.system(a).setup("cptr3-amg", b, max_coarse_size=40)
    for d in (1, -1):
        lg, ng = sg.levelsets(d)
        lo, no = so.levelsets(d)
        assert ng == no and np.array_equal(lg, lo), f"ILU block DAG dir {d}"
    for st in range(2):
        hg, ho = sg.stage_amg(st), so.stage_amg(st)
        for l in range(ho.n_levels - 1):
            for d in (1, -1):
                lg, ng = hg.levelsets(l, d)
                lo, no = ho.levelsets(l, d)
                assert ng == no and np.array_equal(lg, lo), f"stage {st} level {l} dir {d}"


@pytest.mark.parametrize("cid", [1, 2, 3])
def test_levelsets_baseline_configs(gpu, orc, cid):
    from paper_1912_04385_b200 import gen
    a, b, _ = gen.generate(cid)
    method = gen.CONFIG_METHODS[cid][-1]
    sg = gpu.system(a).setup(method, b)
    so = orc.system(a).setup(method, b)
    lg, ng = sg.levelsets(1)
    lo, no = so.levelsets(1)
    nx = int(round(np.sqrt(a.n_cells)))
    assert ng == no == 2 * nx - 1 and np.array_equal(lg, lo)  # square 5-point grid: depth nx + ny - 1
    for st in range(so.n_stages() - 1):
        hg, ho = sg.stage_amg(st), so.stage_amg(st)
        for l in range(ho.n_levels - 1):
            for d in (1, -1):
                lg, ng = hg.levelsets(l, d)
                lo, no = ho.levelsets(l, d)
                assert ng == no and np.array_equal(lg, lo), f"stage {st} level {l} dir {d}"


@pytest.mark.parametrize("name", list(RETRY_SPECS))
def test_retry_loop(gpu, orc, name):
    """solve_system's three attempts (harness.cpp:209-217): the same attempt
    count and convergence verdicts, and per attempt the GPU's iteration counts
    in the oracle's own rounding class.  On g60x60 the counts are chaotic: a
    1e-15 perturbation of b moves the oracle's first attempt over 88..102
    (tests/ensemble.py, scripts/retry_dist.py), so single runs are compared by
    distribution -- both sides solve the same 12 perturbed right-hand sides; the
    per-attempt means agree within 10 % and the ranges overlap."""
    a, b, xs, method = retry_system(name)
    rg = gpu.system(a).setup(method, b, max_coarse_size=40).solve()
    ro = orc.system(a).setup(method, b, max_coarse_size=40).solve()
    assert ro.attempts == 3
    assert rg.attempts == ro.attempts and rg.converged == ro.converged
    assert rg.attempt_converged == ro.attempt_converged
    for tg, to in zip(rg.attempt_true_residual, ro.attempt_true_residual):
        assert (tg <= 1e-8) == (to <= 1e-8)
    gi = [rg.attempt_iterations] + [gpu.system(a).setup(method, perturbed(b, s), max_coarse_size=40).solve()
                                    .attempt_iterations for s in range(12)]
    oi = [ro.attempt_iterations] + [orc.system(a).setup(method, perturbed(b, s), max_coarse_size=40).solve()
                                    .attempt_iterations for s in range(12)]
    gi, oi = np.array([g for g in gi if len(g) == 3]), np.array([o for o in oi if len(o) == 3])
    assert len(gi) >= 10 and len(oi) >= 10
    for q in range(3):
        mg, mo = gi[:, q].mean(), oi[:, q].mean()
        assert abs(mg - mo) <= 0.1 * mo + 1, (q, gi[:, q], oi[:, q])
        assert gi[:, q].min() <= oi[:, q].max() + 1 and oi[:, q].min() <= gi[:, q].max() + 1, (q, gi[:, q], oi[:, q])


def _bad_diag(name, nb, rows_cols, cell):
    a, b, _ = small_system(name)
    vals = a.values.reshape(-1, nb, nb).copy()  # [k][col][row]
    d = a.row_ptr[cell] + int(np.searchsorted(a.col_idx[a.row_ptr[cell]:a.row_ptr[cell + 1]], cell))
    for (r, c) in rows_cols:
        vals[d, c, r] = 0.0
    return BlockMatrix(a.n_cells, nb, a.row_ptr, a.col_idx, vals.reshape(-1)), b


@pytest.mark.parametrize("method,tag", [("cpr-amg", "D_hh"), ("cptr3-amg", "D_ss"), ("cptr-direct", "D_ss")])
def test_singular_block_errors(gpu, orc, method, tag):
    """SingularBlockError{cell_id} tagged with the failing D factor
    (scaling.cpp:40-41): a zero s column in the diagonal block of cell 17."""
    bad, b = _bad_diag("g12x10_nb4_band", 4, [(r, 0) for r in range(4)], 17)
    errs = []
    for api in (gpu, orc):
        with pytest.raises(SingularBlockError) as e:
            api.system(bad).setup(method, b)
        errs.append((e.value.cell_id, str(e.value)))
    assert errs[0] == errs[1] == (17, f"singular {tag} block in cell 17")


def test_singular_d_pp(gpu, orc):
    """CPTR3's second scaling: D_PP = 0 in cell 9 (scaling.cpp:130-136); nb = 2
    so the first scaling leaves the (P,P) entry untouched."""
    from paper_1912_04385_b200 import gen
    a, b, _ = gen.generate(gen.make_spec(6, 5, 2, kappa=1.0, perm_sigma=0.0, band=False, seed=3))
    vals = a.values.reshape(-1, 2, 2).copy()
    d = a.row_ptr[9] + int(np.searchsorted(a.col_idx[a.row_ptr[9]:a.row_ptr[10]], 9))
    vals[d, 0, 0] = 0.0
    bad = BlockMatrix(a.n_cells, 2, a.row_ptr, a.col_idx, vals.reshape(-1))
    errs = []
    for api in (gpu, orc):
        with pytest.raises(SingularBlockError) as e:
            api.system(bad).setup("cptr3-amg", b)
        errs.append((e.value.cell_id, str(e.value)))
    assert errs[0] == errs[1] == (9, "singular D_PP block in cell 9")


def test_dense_factor_pivot_error(gpu, orc):
    """DenseFactor::factor (dense_factor.cpp:12-17): a singular coarsest operator
    raises SingularBlockError(pivot row, "dense-factor pivot")."""
    t = [(i, i, 2.0) for i in range(6)] + [(0, 1, 1.0), (1, 0, 4.0)]
    a = ScalarMatrix.from_triplets(6, t)  # row 1 = 2 * row 0: singular
    errs = []
    for api in (gpu, orc):
        with pytest.raises(SingularBlockError) as e:
            api.amg(a)
        errs.append((e.value.cell_id, str(e.value)))
    assert errs[0] == errs[1]
    assert "dense-factor pivot" in errs[0][1]


def test_amg_stagnation_setup_error(gpu, orc):
    """AMGHierarchy::setup throws when coarsening keeps > 95% of the points
    (amg.cpp:202-204): a one-sided chain makes every point but the first C."""
    n = 1200
    t = [(i, i, 2.0) for i in range(n)] + [(i, i + 1, -1.0) for i in range(n - 1)]
    a = ScalarMatrix.from_triplets(n, t)
    msgs = []
    for api in (gpu, orc):
        with pytest.raises(SetupError) as e:
            api.amg(a)
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1] == "AMG coarsening stagnated at size 1200"


def test_zero_rhs_solve_system(gpu, orc):
    """b = 0: converged with x = 0 (gmres.cpp:17-21) on a fresh handle."""
    a, b, _ = small_system("g12x10_nb4_band")
    z = np.zeros_like(b)
    for api in (gpu, orc):
        r = api.system(a).setup("cptr3-amg", z).solve()
        assert r.converged and r.iterations == 0 and not np.any(r.x)


def test_stale_amg_view_after_resetup(gpu):
    """A re-setup invalidates earlier stage views: they report SetupError
    instead of touching freed hierarchies."""
    a, b, _ = small_system("g12x10_nb4_band")
    s = gpu.system(a).setup("cptr3-amg", b, max_coarse_size=40)
    h = s.stage_amg(0)
    assert h.n_levels >= 1
    s.setup("cpr-amg", b, max_coarse_size=40)
    with pytest.raises(SetupError):
        h.n_levels
    assert s.stage_amg(0).n_levels >= 1


def test_gmres_rejects_mismatched_ilu(gpu):
    a, b, _ = small_system("g12x10_nb4_band")
    small, _, _ = small_system("g8x6_nb3")
    f = gpu.ilu0(small)
    with pytest.raises(DimensionError):
        gpu.gmres(a, b, f)


@pytest.mark.parametrize("name", ["g30x30_nb5_loPe", "g16x16_nb8_band"])
def test_setup_is_reproducible(gpu, name):
    """Two setups of the same system give bitwise identical solves: the sweep
    kernel choice is a fixed rule, not a timing race."""
    a, b, _ = small_system(name)
    runs = [gpu.system(a).setup("cptr3-amg", b, max_coarse_size=40).solve() for _ in range(2)]
    assert runs[0].iterations == runs[1].iterations
    assert np.array_equal(runs[0].residual_history, runs[1].residual_history)
    assert np.array_equal(runs[0].x, runs[1].x)


def test_direct_methods_apply(gpu, orc):
    a, b, _ = small_system("g12x10_nb4_band")
    r = random_vec(a.dim, 7)
    for m in ("cpr-direct", "cptr-direct", "cptr3-direct", "ilu0"):
        sg, so = gpu.system(a).setup(m, b), orc.system(a).setup(m, b)
        assert rel(sg.apply(r), so.apply(r)) < 1e-10, m
        assert isinstance(sg.solve(), SolveResult)
