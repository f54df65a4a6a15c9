"""Known-answer tests of the reference, ported (proj/tests/test_subprec.cpp,
test_krylov.cpp, test_stages.cpp, acceptance.cpp criteria 3/4/6/7).

Every test runs against the CPU oracle (pinning the oracle to the
reference's own expectations) and, under -m gpu, against the sm_100a library
through the identical C ABI.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from paper_1912_04385_b200.api import (BlockMatrix, ConfigError, ScalarMatrix, SetupError, ZeroPivotError,
                                       method_name, parse_method)
from tests.systems import (laplacian_1d, laplacian_2d, random_block_system, random_nonsymmetric, random_vec,
                           small_system)


@pytest.fixture(params=["orc", "ref", pytest.param("gpu", marks=pytest.mark.gpu)])
def api(request):
    return request.getfixturevalue(request.param)


def dense(m: ScalarMatrix) -> np.ndarray:
    return m.to_dense()


def csr(rp, ci, v, shape):
    return sp.csr_matrix((v, ci, rp), shape=shape)


# ------------------------------------------------------------ ILU(0) -------
# test_subprec.cpp:75-134

def test_ilu_diagonal_is_exact(api):
    a = ScalarMatrix.from_triplets(3, [(0, 0, 2.0), (1, 1, 4.0), (2, 2, 8.0)])
    f = api.ilu0(a)
    assert np.array_equal(f.factors(), a.values)
    r = random_vec(3, 1)
    assert np.linalg.norm(f.apply(r) - r / np.array([2.0, 4.0, 8.0])) < 1e-15


def _lu_product(n, rp, ci, v):
    d = csr(rp, ci, v, (n, n)).toarray()
    lower = np.tril(d, -1) + np.eye(n)
    upper = np.triu(d)
    return lower @ upper


def test_ilu_tridiagonal_is_exact_factorization(api):
    a = laplacian_1d(12)
    f = api.ilu0(a)
    lu = _lu_product(12, a.row_ptr, a.col_idx, f.factors())
    assert np.linalg.norm(dense(a) - lu) < 1e-12
    r = random_vec(12, 2)
    x = f.apply(r)
    assert np.linalg.norm(dense(a) @ x - r) / np.linalg.norm(r) < 1e-12


def test_ilu_residual_vanishes_on_pattern(api):
    a = laplacian_2d(8)
    f = api.ilu0(a)
    err = dense(a) - _lu_product(a.n, a.row_ptr, a.col_idx, f.factors())
    for i in range(a.n):
        for k in range(a.row_ptr[i], a.row_ptr[i + 1]):
            assert abs(err[i, a.col_idx[k]]) < 1e-13


def _dense_ilu0(a: ScalarMatrix):
    n = a.n
    lu = dense(a)
    pat = np.zeros((n, n), bool)
    for i in range(n):
        pat[i, a.col_idx[a.row_ptr[i]:a.row_ptr[i + 1]]] = True
    for i in range(1, n):
        for k in range(i):
            if not pat[i, k]:
                continue
            lu[i, k] /= lu[k, k]
            for j in range(k + 1, n):
                if pat[i, j]:
                    lu[i, j] -= lu[i, k] * lu[k, j]
    return lu


def test_ilu_matches_dense_pattern_restricted_elimination(api):
    rng = np.random.default_rng(7)
    n, t = 30, []
    for i in range(n):
        t.append((i, i, 10.0 + rng.uniform(-1, 1)))
        for _ in range(4):
            j = int(rng.integers(n))
            if j != i:
                t.append((i, j, rng.uniform(-1, 1)))
    a = ScalarMatrix.from_triplets(n, t)
    f = api.ilu0(a).factors()
    ref = _dense_ilu0(a)
    for i in range(n):
        for k in range(a.row_ptr[i], a.row_ptr[i + 1]):
            j = a.col_idx[k]
            assert f[k] == pytest.approx(ref[i, j], rel=1e-12, abs=1e-14)


def test_ilu_rejects_zero_pivot(api):
    a = ScalarMatrix.from_triplets(2, [(0, 0, 1.0), (0, 1, 1.0), (1, 0, 2.0), (1, 1, 2.0)])
    with pytest.raises(ZeroPivotError) as e:
        api.ilu0(a)
    assert e.value.row_id == 1


def test_ilu_rejects_missing_diagonal(api):
    a = ScalarMatrix.from_triplets(2, [(0, 1, 1.0), (1, 0, 1.0), (1, 1, 1.0)])
    with pytest.raises(SetupError):
        api.ilu0(a)


def test_block_ilu_equals_scalar_ilu(orc):
    """Block restatement == line-for-line scalar ILU0Factor on the flattening."""
    import ctypes as C
    for name in ["g8x6_nb3", "g12x10_nb4_band"]:
        a, _, _ = small_system(name)
        blk = orc.ilu0(a).factors()
        flat = np.zeros(a.values.size)
        orc.check(orc.lib.orc_ilu_scalar_factor(C.byref(a._c), flat.ctypes.data))
        # flat CSR order: per scalar row, blocks ascending, columns ascending
        nb = a.nb
        exp = np.empty_like(flat)
        o = 0
        b = blk.reshape(-1, nb, nb).transpose(0, 2, 1)  # [k][r][c]
        for cell in range(a.n_cells):
            for r in range(nb):
                for k in range(a.row_ptr[cell], a.row_ptr[cell + 1]):
                    exp[o:o + nb] = b[k, r, :]
                    o += nb
        assert np.array_equal(exp, flat)
        r = random_vec(a.dim, 3)
        y_scalar = np.zeros(a.dim)
        orc.check(orc.lib.orc_ilu_scalar_apply(C.byref(a._c), r.ctypes.data, y_scalar.ctypes.data))
        assert np.array_equal(orc.ilu0(a).apply(r), y_scalar)


# ------------------------------------------------------------------- AMG ---
# test_subprec.cpp:149-202

def test_amg_single_exact_level_below_cutoff(api):
    a = laplacian_2d(5)
    h = api.amg(a)
    assert h.n_levels == 1
    r = random_vec(25, 5)
    assert np.linalg.norm(dense(a) @ h.apply(r) - r) / np.linalg.norm(r) < 1e-12


def test_coarsening_halves_a_1d_chain(api):
    a = laplacian_1d(64)
    h = api.amg(a, max_coarse_size=32)
    assert h.n_levels == 2
    cf = h.cf(0)
    assert int(cf.sum()) == 32
    n1, _, _ = h.level_info(1)
    assert n1 == 32
    rp, ci, v = h.level_csr(1, 1)
    p = csr(rp, ci, v, (64, 32))
    interp = p @ np.ones(32)
    assert np.allclose(interp[1:63], 1.0, rtol=1e-13, atol=1e-13)


def test_amg_galerkin_products_on_64x64(api):
    a = laplacian_2d(64)
    h = api.amg(a)
    assert h.n_levels >= 2
    assert h.level_info(h.n_levels - 1)[0] <= 1000
    prev = csr(a.row_ptr, a.col_idx, a.values, (a.n, a.n))
    for l in range(1, h.n_levels):
        n, _, _ = h.level_info(l)
        nf = prev.shape[0]
        p = csr(*h.level_csr(l, 1), (nf, n))
        r = csr(*h.level_csr(l, 2), (n, nf))
        ac = csr(*h.level_csr(l, 0), (n, n))
        rap = r @ (prev @ p)
        assert abs(r - p.T).max() == 0
        assert sp.linalg.norm(ac - rap) / sp.linalg.norm(ac) < 1e-13
        prev = ac


def test_one_vcycle_halves_the_residual(api):
    a = laplacian_2d(32)
    h = api.amg(a, max_coarse_size=40)
    b = random_vec(a.n, 6)
    x = h.apply(b)
    assert np.linalg.norm(b - dense(a) @ x) / np.linalg.norm(b) <= 0.5


def test_amg_maps_zero_to_zero(api):
    a = laplacian_2d(16)
    h = api.amg(a, max_coarse_size=20)
    assert np.linalg.norm(h.apply(np.zeros(a.n))) == 0.0


# ----------------------------------------------------------------- GMRES ---
# test_krylov.cpp:46-149

def _identity(n):
    return ScalarMatrix(n, np.arange(n + 1), np.arange(n), np.ones(n))


def test_identity_converges_in_one_iteration(api):
    b = random_vec(20, 1)
    r = api.gmres(_identity(20), b)
    assert r.converged and r.iterations == 1
    assert np.linalg.norm(r.x - b) < 1e-14


def test_unpreconditioned_within_dim_and_matches_dense(api):
    a = random_nonsymmetric(40, 2)
    b = random_vec(40, 3)
    r = api.gmres(a, b, tol=1e-10, max_iter=200)
    assert r.converged and r.iterations <= 40
    x_ref = np.linalg.solve(dense(a), b)
    assert np.linalg.norm(r.x - x_ref) / np.linalg.norm(x_ref) < 1e-6
    assert r.final_true_residual < 1e-8


def test_exact_inverse_preconditioner_one_iteration(api):
    """ILU(0) on a full pattern is the exact LU: an exact inverse preconditioner."""
    rng = np.random.default_rng(5)
    n = 25
    d = rng.uniform(-1, 1, (n, n)) + 6.0 * np.eye(n)
    a = ScalarMatrix(n, np.arange(n + 1) * n, np.tile(np.arange(n), n), d.reshape(-1))
    m = api.ilu0(a)
    b = random_vec(n, 7)
    r = api.gmres(a, b, prec=m)
    assert r.converged and r.iterations == 1
    assert r.final_true_residual < 1e-10


def test_residual_history_monotone(api):
    a = laplacian_1d(60)
    r = api.gmres(a, random_vec(60, 11), tol=1e-10, max_iter=200)
    assert r.converged and len(r.residual_history) >= 2
    h = r.residual_history
    assert np.all(h[1:] <= h[:-1] + 1e-10)
    assert h[-1] <= 1e-10


def test_repeated_solves_bitwise_deterministic(api):
    a = random_nonsymmetric(30, 13)
    b = random_vec(30, 17)
    r1, r2 = api.gmres(a, b), api.gmres(a, b)
    assert r1.iterations == r2.iterations
    assert np.array_equal(r1.x, r2.x)
    assert np.array_equal(r1.residual_history, r2.residual_history)


def test_zero_rhs_returns_zero(api):
    r = api.gmres(laplacian_1d(10), np.zeros(10))
    assert r.converged and np.linalg.norm(r.x) == 0.0


def test_iteration_cap_reports_non_convergence(api):
    r = api.gmres(laplacian_1d(100), random_vec(100, 29), tol=1e-14, max_iter=5)
    assert not r.converged and r.iterations == 5 and r.final_true_residual > 1e-14


@pytest.mark.parametrize("n", [30, 60, 120])
def test_acceptance_6_unpreconditioned_within_n(api, n):
    a = random_nonsymmetric(n, 600 + n, diag=8.0)
    r = api.gmres(a, random_vec(n, 650 + n), tol=1e-8, max_iter=2 * n)
    assert r.converged and r.iterations <= n and r.final_true_residual <= 1e-8


def test_acceptance_7_amg_scalability(api):
    prev = 0
    for n in (32, 64, 128):
        a = laplacian_2d(n)
        h = api.amg(a, max_coarse_size=100)
        r = api.gmres(a, random_vec(a.n, 700 + n), prec=h, tol=1e-8, max_iter=100)
        assert r.converged
        if n == 128:
            assert r.iterations <= 25
        if prev:
            assert r.iterations <= int(np.ceil(1.3 * prev))
        prev = r.iterations


# -------------------------------------------------------- scaling/stages ---
# test_stages.cpp:93-272

def test_method_names():
    for name in ("ilu0", "cpr-direct", "cpr-amg", "cptr-direct", "cptr3-direct", "cptr3-amg"):
        assert method_name(parse_method(name)) == name
    with pytest.raises(ConfigError):
        parse_method("cptr-amg")
    with pytest.raises(ConfigError):
        parse_method("gmres")


def _scaling_oracle(a: BlockMatrix, method: str) -> np.ndarray:
    """Dense N^-1 = E (test_stages.cpp:36-66)."""
    nb, n = a.nb, a.dim
    ns = nb - 2
    e = np.eye(n)
    blocks = a.blocks()
    for c in range(a.n_cells):
        k = [k for k in range(a.row_ptr[c], a.row_ptr[c + 1]) if a.col_idx[k] == c][0]
        d = blocks[k]
        off = c * nb
        if method == "cpr":
            h = list(range(ns)) + [ns + 1]
            w = d[ns, h] @ np.linalg.inv(d[np.ix_(h, h)])
            for i, hi in enumerate(h):
                e[off + ns, off + hi] -= w[i]
        else:
            w = d[ns:ns + 2, :ns] @ np.linalg.inv(d[:ns, :ns])
            for r in range(2):
                for k2 in range(ns):
                    e[off + ns + r, off + k2] -= w[r, k2]
    return e


@pytest.mark.parametrize("seed", [3, 5])
def test_cpr_scaling_matches_dense_oracle(api, seed):
    a = random_block_system(4, 3, seed)
    b = random_vec(a.dim, seed + 100)
    s = api.system(a).setup("cpr-amg", b)
    abar, bbar = s.scaled()
    e = _scaling_oracle(a, "cpr")
    want = e @ a.to_dense()
    got = BlockMatrix(a.n_cells, a.nb, a.row_ptr, a.col_idx, abar).to_dense()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-13
    assert np.linalg.norm(bbar - e @ b) / np.linalg.norm(b) < 1e-13
    x = np.linalg.solve(a.to_dense(), b)
    assert np.linalg.norm(got @ x - bbar) / np.linalg.norm(bbar) < 1e-12
    ns = a.nb - 2
    for c in range(a.n_cells):
        k = [k for k in range(a.row_ptr[c], a.row_ptr[c + 1]) if a.col_idx[k] == c][0]
        d = got[c * a.nb:(c + 1) * a.nb, c * a.nb:(c + 1) * a.nb]
        scale = np.linalg.norm(a.blocks()[k])
        assert np.all(np.abs(d[ns, :ns]) < 1e-13 * scale) and abs(d[ns, ns + 1]) < 1e-13 * scale


def test_cptr3_scaling_equals_two_step_dense(api):
    a = random_block_system(3, 3, 7)
    b = random_vec(a.dim, 8)
    nb = a.nb
    e1 = _scaling_oracle(a, "cptr")
    once = e1 @ a.to_dense()
    e2 = np.eye(a.dim)
    for c in range(a.n_cells):
        p, t = c * nb + nb - 2, c * nb + nb - 1
        e2[t, p] = -once[t, p] / once[p, p]
    want = e2 @ once
    s = api.system(a).setup("cptr3-amg", b)
    abar, bbar = s.scaled()
    got = BlockMatrix(a.n_cells, nb, a.row_ptr, a.col_idx, abar).to_dense()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-13
    assert np.linalg.norm(bbar - e2 @ (e1 @ b)) / np.linalg.norm(b) < 1e-13


def _densify(n, op):
    return np.column_stack([op(np.eye(n)[:, j]) for j in range(n)])


@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg", "cpr-direct", "cptr-direct", "cptr3-direct"])
def test_stage_composition_equals_explicit(api, method):
    """Alg. 1/2 == M1 + M2(I - A M1) [+ M3(I - A M2)(I - A M1)]."""
    a = random_block_system(4, 2, 11)
    n = a.dim
    s = api.system(a).setup(method, random_vec(n, 12))
    abar = BlockMatrix(a.n_cells, a.nb, a.row_ptr, a.col_idx, s.scaled()[0]).to_dense()
    ms = [_densify(n, lambda v, i=i: s.apply_stage(i, v)) for i in range(s.n_stages())]
    eye = np.eye(n)
    if len(ms) == 2:
        comp = ms[0] + ms[1] @ (eye - abar @ ms[0])
    else:
        comp = ms[0] + ms[1] @ (eye - abar @ ms[0]) + ms[2] @ (eye - abar @ ms[1]) @ (eye - abar @ ms[0])
    r = random_vec(n, 19)
    via = s.apply(r)
    assert np.linalg.norm(via - comp @ r) / np.linalg.norm(via) < 1e-13


def test_stage_counts_and_scopes(api):
    a = random_block_system(4, 2, 23)
    b = random_vec(a.dim, 1)
    assert api.system(a).setup("cpr-amg", b).n_stages() == 2
    assert api.system(a).setup("cptr3-amg", b).n_stages() == 3
    assert api.system(a).setup("ilu0", b).n_stages() == 1
    s = api.system(a).setup("cptr3-amg", b)
    r = random_vec(a.dim, 2)
    y0, y1 = s.apply_stage(0, r), s.apply_stage(1, r)
    nb = a.nb
    mask_t = np.zeros(a.dim, bool)
    mask_t[nb - 1::nb] = True
    mask_p = np.zeros(a.dim, bool)
    mask_p[nb - 2::nb] = True
    assert np.all(y0[~mask_t] == 0) and np.all(y1[~mask_p] == 0)


@pytest.mark.parametrize("method", ["ilu0", "cpr-direct", "cptr-direct", "cptr3-direct", "cptr3-amg"])
def test_preconditioners_linear_and_zero(api, method):
    a = random_block_system(3, 3, 29)
    s = api.system(a).setup(method, random_vec(a.dim, 1))
    assert np.linalg.norm(s.apply(np.zeros(a.dim))) == 0.0
    r1, r2 = random_vec(a.dim, 31), random_vec(a.dim, 37)
    lin = s.apply(2.0 * r1 - 0.5 * r2)
    parts = 2.0 * s.apply(r1) - 0.5 * s.apply(r2)
    assert np.linalg.norm(lin - parts) / (1.0 + np.linalg.norm(parts)) < 1e-13


def test_ilu0_baseline_equals_direct_factor(api):
    a = random_block_system(3, 3, 41)
    s = api.system(a).setup("ilu0", random_vec(a.dim, 1))
    r = random_vec(a.dim, 43)
    assert np.array_equal(s.apply(r), api.ilu0(a).apply(r))


@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg"])
def test_acceptance_4_scaling_preserves_solution(api, method):
    a, b, xs = small_system("g12x10_nb4_band")
    s = api.system(a).setup(method, b)
    abar, bbar = s.scaled()
    xbar = np.linalg.solve(BlockMatrix(a.n_cells, a.nb, a.row_ptr, a.col_idx, abar).to_dense(), bbar)
    x = np.linalg.solve(a.to_dense(), b)
    assert np.linalg.norm(xbar - x) / np.linalg.norm(x) < 1e-12


@pytest.mark.parametrize("method", ["cpr-amg", "cptr3-amg"])
def test_solve_system_recovers_xstar(api, method):
    a, b, xs = small_system("g12x10_nb4_band")
    r = api.system(a).setup(method, b).solve()
    assert r.converged and r.final_true_residual <= 1e-8
    assert np.linalg.norm(r.x - xs) / np.linalg.norm(xs) < 1e-6


def test_cptr_scaling_matches_dense_oracle(api):
    """test_stages.cpp:152-162 (B_ee is the elliptic view of the scaled system)."""
    a = random_block_system(4, 3, 5)
    b = random_vec(a.dim, 6)
    s = api.system(a).setup("cptr-direct", b)
    abar, bbar = s.scaled()
    e = _scaling_oracle(a, "cptr")
    want = e @ a.to_dense()
    got = BlockMatrix(a.n_cells, a.nb, a.row_ptr, a.col_idx, abar).to_dense()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) < 1e-13
    assert np.linalg.norm(bbar - e @ b) / np.linalg.norm(b) < 1e-13
    assert s.n_stages() == 2
    r = random_vec(a.dim, 7)
    y0 = s.apply_stage(0, r)
    mask = np.zeros(a.dim, bool)
    mask[a.nb - 2::a.nb] = True
    mask[a.nb - 1::a.nb] = True
    assert np.all(y0[~mask] == 0)  # scope = indices_of(elliptic)


@pytest.mark.parametrize("method", ["cpr-direct", "cptr-direct", "cptr3-direct"])
def test_preconditioned_solution_matches_unscaled(api, method):
    """test_krylov.cpp:119-139: direct methods, tol 1e-12, x vs the dense solve."""
    a = random_block_system(5, 3, 23)
    b = random_vec(a.dim, 24)
    x_ref = np.linalg.solve(a.to_dense(), b)
    r = api.system(a).setup(method, b).solve(tol=1e-12, max_iter=200)
    assert r.converged
    assert np.linalg.norm(r.x - x_ref) / np.linalg.norm(x_ref) < 1e-8


def test_acceptance_5_direct_methods_exact_on_decoupled_fields(api):
    """acceptance.cpp:193-226: fields mutually decoupled, tridiagonal chains per
    field -> every -direct method converges in exactly one iteration."""
    rng = np.random.default_rng(505)
    n_cells, blocks = 20, {}
    for c in range(n_cells):
        blocks[(c, c)] = np.diag(3.0 + rng.uniform(0.1, 0.9, 3))
        if c + 1 < n_cells:
            blocks[(c, c + 1)] = np.diag(-rng.uniform(0.1, 0.9, 3))
            blocks[(c + 1, c)] = np.diag(-rng.uniform(0.1, 0.9, 3))
    a = BlockMatrix.from_dense_blocks(n_cells, 3, blocks)
    b = random_vec(a.dim, 42)
    for method in ("cpr-direct", "cptr-direct", "cptr3-direct"):
        r = api.system(a).setup(method, b).solve()
        assert r.converged and r.iterations == 1, (method, r.iterations)


def test_acceptance_3_compositions_on_random_systems(api):
    """acceptance.cpp:120-167 (10 systems here): staged applications equal the
    explicit compositions with -direct sub-solvers."""
    worst = 0.0
    for trial in range(10):
        a = random_block_system(2 + trial % 7, 3, 700 + trial)
        n = a.dim
        r = random_vec(n, 800 + trial)
        for method in ("cpr-direct", "cptr3-direct"):
            s = api.system(a).setup(method, random_vec(n, 1))
            abar = BlockMatrix(a.n_cells, a.nb, a.row_ptr, a.col_idx, s.scaled()[0]).to_dense()
            ms = [_densify(n, lambda v, i=i: s.apply_stage(i, v)) for i in range(s.n_stages())]
            eye = np.eye(n)
            if len(ms) == 2:
                comp = (ms[0] + ms[1] @ (eye - abar @ ms[0])) @ r
            else:
                comp = (ms[0] + ms[1] @ (eye - abar @ ms[0]) + ms[2] @ (eye - abar @ ms[1]) @ (eye - abar @ ms[0])) @ r
            worst = max(worst, np.linalg.norm(s.apply(r) - comp) / (1.0 + np.linalg.norm(comp)))
    assert worst <= 1e-13, worst
