"""Static condensation (condense.cpp:206-258).

CPU tests pin the oracle with the reference's own known-answer tests
(proj/tests/test_condense.cpp, acceptance.cpp:69-95 criterion 1); GPU tests
hold the device condensation to the oracle bitwise (A, b, the secondary
update) and drive the reduced system through the solver.
"""
import numpy as np
import pytest

from paper_1912_04385_b200 import api as A
from paper_1912_04385_b200 import condense as cd

NAMES = {cd.PRESSURE: "P", cd.TEMPERATURE: "T", cd.GAS_SAT: "Sg", cd.OIL_SAT: "So"}


def names(labels):
    out = []
    for k, i in labels:
        if k == cd.VAPOR_FRAC:
            out.append(f"y{i}")
        elif k == cd.OIL_FRAC:
            out.append(f"x{i}")
        elif k == cd.SOLID:
            out.append(f"c{i}")
        else:
            out.append(NAMES[k])
    return out


# ---- orderings (test_condense.cpp:46-110) -----------------------------------
def test_ordering_sizes():
    for s in cd.STATES:
        vp = cd.ordering_for(s, 12, 1)
        assert vp.n_primary == 14
        assert len(vp.equations) == vp.n_secondary
        assert len(vp.canonical_perm) == 14
    assert [cd.ordering_for(s, 12, 1).n_secondary for s in cd.STATES] == [1, 13, 14]


def test_ordering_lists():
    g = cd.ordering_for("G", 12, 1)
    assert names(g.primary) == ["P"] + [f"y{i}" for i in range(2, 13)] + ["c0", "T"]
    assert names(g.secondary) == ["y1"]
    og = cd.ordering_for("OG", 12, 1)
    assert names(og.primary) == ["P", "Sg", "y3"] + [f"x{i}" for i in range(4, 13)] + ["c0", "T"]
    assert names(og.secondary) == ["y1", "x2"] + [f"y{i}" for i in range(4, 13)] + ["y2", "x1"]
    owg = cd.ordering_for("OWG", 12, 1)
    assert names(owg.primary) == ["P", "Sg", "So"] + [f"x{i}" for i in range(4, 13)] + ["c0", "T"]
    assert names(owg.secondary) == ["y1", "x2", "y3"] + [f"y{i}" for i in range(4, 13)] + ["y2", "x3"]


def test_canonical_perm_ends_with_p_t():
    for s in cd.STATES:
        vp = cd.ordering_for(s, 12, 1)
        assert vp.primary[vp.canonical_perm[-2]][0] == cd.PRESSURE
        assert vp.primary[vp.canonical_perm[-1]][0] == cd.TEMPERATURE
        assert sorted(vp.canonical_perm) == list(range(14))


def test_secondary_diagonals_nonzero():
    rng = np.random.default_rng(5)
    for t in range(100):
        vp = cd.ordering_for(cd.STATES[t % 3], 12, 1)
        j22, _, _ = cd.make_cell_secondary_blocks(vp, rng)
        assert np.all(np.diag(j22) != 0.0)


# ---- oracle against the dense full-system solve -----------------------------
def _check_reduced_solve(api, j, tol=1e-10):
    red = api.condense(j)
    d1 = np.linalg.solve(red.a.to_dense(), red.b)
    d2 = red.back_substitute(d1)
    J, mr = j.to_dense_full()
    ref = np.linalg.solve(J, mr)
    x = np.concatenate([d1, d2])
    return np.linalg.norm(x - ref) / np.linalg.norm(ref)


def test_criterion_1_oracle(orc):
    """acceptance.cpp:69-95: 25 systems of 2-20 cells, n_c=12, n_s=1, <= 1e-10."""
    worst = 0.0
    for trial in range(25):
        n = 2 + int(np.random.default_rng(101 + trial).integers(0, 19))
        j = cd.make_synthetic_global(cd.mixed_states(n, 300 + trial), 12, 1, 500 + trial)
        worst = max(worst, _check_reduced_solve(orc, j))
    assert worst <= 1e-10


def test_zero_coupling(orc):
    """test_condense.cpp:144-156."""
    j = cd.make_synthetic_global(cd.mixed_states(3, 7), 12, 1, 4)
    j.j12 = [(r, c, np.zeros_like(b)) for (r, c, b) in j.j12]
    j.j21 = [np.zeros_like(m) for m in j.j21]
    red = orc.condense(j)
    assert np.array_equal(red.a.to_dense(), A.BlockMatrix(j.n_cells, j.np, j.row_ptr, j.col_idx,
                                                           np.concatenate([b.T.reshape(-1) for b in j.j11_blocks])).to_dense())
    assert np.array_equal(red.b, -j.r1)
    j.r2 = [np.zeros_like(v) for v in j.r2]
    red0 = orc.condense(j)
    assert np.linalg.norm(red0.back_substitute(np.zeros(red0.a.dim))) == 0.0


def test_scaling_commutes(orc):
    """test_condense.cpp:201-222: row/column scaling of the secondary blocks."""
    j = cd.make_synthetic_global(cd.mixed_states(5, 31), 12, 1, 31)
    s = cd.make_synthetic_global(cd.mixed_states(5, 31), 12, 1, 31)
    rng = np.random.default_rng(77)
    col_s = []
    for c in range(5):
        ns = j.j22[c].shape[0]
        rs, cs = rng.uniform(0.5, 2.0, ns), rng.uniform(0.5, 2.0, ns)
        col_s.append(cs)
        s.j22[c] = rs[:, None] * j.j22[c] * cs[None, :]
        s.j21[c] = rs[:, None] * j.j21[c]
        s.r2[c] = rs * j.r2[c]
    s.j12 = [(r, c, b * col_s[c][None, :]) for (r, c, b) in j.j12]
    r1, r2 = orc.condense(j), orc.condense(s)
    a1, a2 = r1.a.to_dense(), r2.a.to_dense()
    assert np.linalg.norm(a1 - a2) / np.linalg.norm(a1) < 1e-12
    assert np.linalg.norm(r1.b - r2.b) / np.linalg.norm(r1.b) < 1e-12


def test_singular_secondary_block(orc):
    """test_condense.cpp:224-233: the failing cell is reported."""
    j = cd.make_synthetic_global(cd.mixed_states(4, 41), 12, 1, 41)
    j.j22[3] = np.zeros_like(j.j22[3])
    with pytest.raises(A.SingularBlockError) as e:
        orc.condense(j)
    assert e.value.cell_id == 3


def test_dims(orc):
    """test_condense.cpp:188-199."""
    assert orc.condense(cd.make_synthetic_global(cd.mixed_states(100, 23), 12, 1, 23)).a.dim == 1400
    red = orc.condense(cd.make_synthetic_global(["G"] * 5, 12, 1, 17))
    assert red.back_substitute(np.linalg.solve(red.a.to_dense(), red.b)).size == 5


# ---- GPU: bitwise against the oracle -----------------------------------------
def _pair(gpu, orc, j):
    return gpu.condense(j), orc.condense(j)


@pytest.mark.gpu
@pytest.mark.parametrize("n,seed,coupling", [(2, 1, True), (7, 2, True), (20, 3, True), (12, 4, False),
                                             (150, 5, True)])
def test_gpu_condense_bitwise(gpu, orc, n, seed, coupling):
    j = cd.make_synthetic_global(cd.mixed_states(n, seed), 12, 1, 900 + seed, coupling)
    rg, ro = _pair(gpu, orc, j)
    assert np.array_equal(rg.a.row_ptr, ro.a.row_ptr) and np.array_equal(rg.a.col_idx, ro.a.col_idx)
    assert np.array_equal(rg.a.values, ro.a.values), np.abs(rg.a.values - ro.a.values).max()
    assert np.array_equal(rg.b, ro.b)
    d1 = np.random.default_rng(seed).standard_normal(rg.a.dim)
    assert np.array_equal(rg.back_substitute(d1), ro.back_substitute(d1))


@pytest.mark.gpu
@pytest.mark.parametrize("n_c,n_s", [(3, 0), (6, 2), (20, 1)])
def test_gpu_condense_sizes(gpu, orc, n_c, n_s):
    j = cd.make_synthetic_global(cd.mixed_states(9, n_c), n_c, n_s, 40 + n_c)
    rg, ro = _pair(gpu, orc, j)
    assert np.array_equal(rg.a.values, ro.a.values) and np.array_equal(rg.b, ro.b)


@pytest.mark.gpu
def test_gpu_singular_cell(gpu):
    j = cd.make_synthetic_global(cd.mixed_states(6, 41), 12, 1, 41)
    j.j22[4] = np.zeros_like(j.j22[4])
    j.j22[2] = np.zeros_like(j.j22[2])
    with pytest.raises(A.SingularBlockError) as e:
        gpu.condense(j)
    assert e.value.cell_id == 2


@pytest.mark.gpu
def test_gpu_criterion_1(gpu):
    worst = 0.0
    for trial in range(25):
        n = 2 + int(np.random.default_rng(101 + trial).integers(0, 19))
        j = cd.make_synthetic_global(cd.mixed_states(n, 300 + trial), 12, 1, 500 + trial)
        worst = max(worst, _check_reduced_solve(gpu, j))
    assert worst <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["ilu0", "cpr-direct", "cptr3-direct"])
def test_gpu_condense_then_solve(gpu, orc, method):
    """condense -> reduced solve on the device -> back_substitute, against the
    dense full-system solve (the CLI's condensed path, harness.cpp:153-188)."""
    j = cd.make_synthetic_global(cd.mixed_states(40, 8), 12, 1, 808)
    red = gpu.condense(j)
    s = red.system().setup(method)
    r = s.solve(tol=1e-12, max_iter=400)
    d2 = red.back_substitute(r.x)
    J, mr = j.to_dense_full()
    ref = np.linalg.solve(J, mr)
    x = np.concatenate([r.x, d2])
    assert np.linalg.norm(x - ref) / np.linalg.norm(ref) < 1e-8
    so = orc.condense(j).system().setup(method)
    ro = so.solve(tol=1e-12, max_iter=400)
    assert abs(r.iterations - ro.iterations) <= 1
