"""Test systems.  Structures follow the reference's own fixtures
(proj/tests/test_subprec.cpp:14-72, test_krylov.cpp:14-44,
test_blockmat.cpp:14-38); values are numpy-seeded."""
import numpy as np

from paper_1912_04385_b200 import gen
from paper_1912_04385_b200.api import BlockMatrix, ScalarMatrix


def laplacian_1d(n, diag=2.0):
    t = []
    for i in range(n):
        t.append((i, i, diag))
        if i > 0:
            t.append((i, i - 1, -1.0))
        if i + 1 < n:
            t.append((i, i + 1, -1.0))
    return ScalarMatrix.from_triplets(n, t)


def laplacian_2d(n):
    t = []
    idx = lambda i, j: i * n + j  # noqa: E731
    for i in range(n):
        for j in range(n):
            t.append((idx(i, j), idx(i, j), 4.0))
            if i > 0:
                t.append((idx(i, j), idx(i - 1, j), -1.0))
            if i + 1 < n:
                t.append((idx(i, j), idx(i + 1, j), -1.0))
            if j > 0:
                t.append((idx(i, j), idx(i, j - 1), -1.0))
            if j + 1 < n:
                t.append((idx(i, j), idx(i, j + 1), -1.0))
    return ScalarMatrix.from_triplets(n * n, t)


def random_nonsymmetric(n, seed, diag=6.0, per_row=3):
    rng = np.random.default_rng(seed)
    t = []
    for i in range(n):
        t.append((i, i, diag + rng.uniform(-1, 1)))
        for _ in range(per_row):
            j = int(rng.integers(n))
            if j != i:
                t.append((i, j, rng.uniform(-1, 1)))
    return ScalarMatrix.from_triplets(n, t)


def random_vec(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def random_block_system(n_cells, n_s, seed, chain=True):
    """Block tridiagonal chain with a dominant diagonal (test_blockmat.cpp:24-38)."""
    rng = np.random.default_rng(seed)
    m = n_s + 2
    blocks = {}
    for c in range(n_cells):
        d = rng.uniform(-1, 1, (m, m))
        d[np.diag_indices(m)] += 4.0 * m
        blocks[(c, c)] = d
        if chain and c + 1 < n_cells:
            blocks[(c, c + 1)] = rng.uniform(-1, 1, (m, m))
            blocks[(c + 1, c)] = rng.uniform(-1, 1, (m, m))
    return BlockMatrix.from_dense_blocks(n_cells, m, blocks)


# Small members of the BASELINE generator family used for parity sweeps.
SMALL_SPECS = {
    "g8x6_nb3": dict(nx=8, ny=6, nb=3, kappa=1.0, perm_sigma=0.0, band=False, seed=11),
    "g12x10_nb4_band": dict(nx=12, ny=10, nb=4, kappa=1.0, perm_sigma=1.0, band=True, seed=7),
    "g20x20_nb4_hiPe": dict(nx=20, ny=20, nb=4, kappa=1e-3, perm_sigma=2.0, band=False, seed=2),
    "g16x16_nb8_band": dict(nx=16, ny=16, nb=8, kappa=1.0, perm_sigma=1.5, band=True, seed=4),
    "g30x30_nb5_loPe": dict(nx=30, ny=30, nb=5, kappa=1e3, perm_sigma=2.0, band=False, seed=3),
}


def small_system(name):
    return gen.generate(gen.make_spec(**SMALL_SPECS[name]))


# Members of the config-4 family (reaction band, nb = 8) on which solve_system
# needs all three tolerance-tightening attempts (harness.cpp:209-217): the
# scaled residual reaches tol while the true residual does not.
RETRY_SPECS = {
    "g20x20_nb8_band_s1": (dict(nx=20, ny=20, nb=8, kappa=1.0, perm_sigma=1.5, band=True, seed=1), "cptr3-amg"),
    "g60x60_nb8_band_s1": (dict(nx=60, ny=60, nb=8, kappa=1.0, perm_sigma=1.5, band=True, seed=1), "cpr-amg"),
}


def retry_system(name):
    spec, method = RETRY_SPECS[name]
    a, b, xs = gen.generate(gen.make_spec(**spec))
    return a, b, xs, method
