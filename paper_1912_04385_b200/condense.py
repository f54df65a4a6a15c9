"""GlobalJacobian for static condensation (proj/include/mprec/condense.hpp).

`GlobalJacobian` carries the full thermal-compositional Jacobian split into
primary / secondary blocks (condense.hpp:64-81) as flat arrays in the C ABI's
`mprec_global_jacobian` layout; `Api.condense` (api.py) reduces it on the
device.  `make_synthetic_global` restates the reference's synthetic generator
(condense.cpp:359-421) -- the variable partitions of `ordering_for`
(condense.cpp:85-147) and the structural dependency patterns of
`make_cell_secondary_blocks` (condense.cpp:318-356) -- drawing from numpy's
seeded PCG64 instead of std::mt19937_64 (same structure and value
distributions, not the same numbers).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

# ---- variable partition (condense.hpp:44-58, condense.cpp:85-147) -----------
PRESSURE, TEMPERATURE, GAS_SAT, OIL_SAT, VAPOR_FRAC, OIL_FRAC, SOLID = range(7)
FUGACITY, GAS_CONSTRAINT, OIL_CONSTRAINT = range(3)
STATES = ("G", "OG", "OWG")


@dataclass
class VariablePartition:
    state: str
    n_c: int
    n_s: int
    primary: list = field(default_factory=list)    # list order: [flow primary..., solids, T]
    secondary: list = field(default_factory=list)
    equations: list = field(default_factory=list)  # aligned with `secondary`
    canonical_perm: list = field(default_factory=list)

    @property
    def n_primary(self) -> int:
        return len(self.primary)

    @property
    def n_secondary(self) -> int:
        return len(self.secondary)

    def canonical_labels(self) -> list:
        return [self.primary[p] for p in self.canonical_perm]


def ordering_for(state: str, n_c: int, n_s: int) -> VariablePartition:
    """ordering_for (condense.cpp:85-141): primary / secondary unknowns of a cell."""
    if n_c < 3:
        raise ValueError("need at least 3 mobile components")
    if n_s < 0:
        raise ValueError("negative solid species count")
    vp = VariablePartition(state, n_c, n_s)
    P, S = vp.primary, vp.secondary
    E = vp.equations
    P.append((PRESSURE, 0))
    if state == "G":
        P.extend((VAPOR_FRAC, i) for i in range(2, n_c + 1))
        S.append((VAPOR_FRAC, 1))
        E.append((GAS_CONSTRAINT, 0))
    elif state == "OG":
        P += [(GAS_SAT, 0), (VAPOR_FRAC, 3)]
        P.extend((OIL_FRAC, i) for i in range(4, n_c + 1))
        S += [(VAPOR_FRAC, 1), (OIL_FRAC, 2)]
        E += [(FUGACITY, 1), (FUGACITY, 2)]
        for i in range(4, n_c + 1):
            S.append((VAPOR_FRAC, i))
            E.append((FUGACITY, i))
        S += [(VAPOR_FRAC, 2), (OIL_FRAC, 1)]
        E += [(GAS_CONSTRAINT, 0), (OIL_CONSTRAINT, 0)]
    elif state == "OWG":
        P += [(GAS_SAT, 0), (OIL_SAT, 0)]
        P.extend((OIL_FRAC, i) for i in range(4, n_c + 1))
        S += [(VAPOR_FRAC, 1), (OIL_FRAC, 2), (VAPOR_FRAC, 3)]
        E += [(FUGACITY, 1), (FUGACITY, 2), (FUGACITY, 3)]
        for i in range(4, n_c + 1):
            S.append((VAPOR_FRAC, i))
            E.append((FUGACITY, i))
        S += [(VAPOR_FRAC, 2), (OIL_FRAC, 3)]
        E += [(GAS_CONSTRAINT, 0), (OIL_CONSTRAINT, 0)]
    else:
        raise ValueError(f"unknown phase state tag '{state}'")
    P.extend((SOLID, k) for k in range(n_s))
    P.append((TEMPERATURE, 0))
    # canonical order = (everything except P and T, in list order), P, T
    rest = [i for i, l in enumerate(P) if l[0] not in (PRESSURE, TEMPERATURE)]
    vp.canonical_perm = rest + [[l[0] for l in P].index(PRESSURE), [l[0] for l in P].index(TEMPERATURE)]
    return vp


def _counterpart(l):
    return (OIL_FRAC, l[1]) if l[0] == VAPOR_FRAC else (VAPOR_FRAC, l[1])


class _GJ(C.Structure):
    _fields_ = [("n_cells", C.c_int), ("np", C.c_int), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("j11", C.c_void_p), ("sec_off", C.c_void_p), ("j22", C.c_void_p), ("j21", C.c_void_p),
                ("n_j12", C.c_int), ("j12_row", C.c_void_p), ("j12_col", C.c_void_p), ("j12", C.c_void_p),
                ("r1", C.c_void_p), ("r2", C.c_void_p)]


class GlobalJacobian:
    """GlobalJacobian (condense.hpp:64-81) with uniform np x np primary blocks.

    j11: (row_ptr, col_idx, blocks (nnzb, np, np)); j22[c]: (ns, ns); j21[c]:
    (ns, np); j12: list of (cell_row, cell_col, (np, ns_col)); r1: (n_cells*np,);
    r2[c]: (ns,).  All matrices row-major numpy here; packed column-major for
    the C ABI."""

    def __init__(self, n_cells, np_, row_ptr, col_idx, j11_blocks, j22, j21, j12, r1, r2, partitions=None):
        self.n_cells, self.np = int(n_cells), int(np_)
        self.row_ptr = np.ascontiguousarray(row_ptr, np.int32)
        self.col_idx = np.ascontiguousarray(col_idx, np.int32)
        self.j11_blocks = np.asarray(j11_blocks, float).reshape(-1, self.np, self.np)
        self.j22 = [np.asarray(m, float).reshape(len(m), -1) if len(m) else np.zeros((0, 0)) for m in j22]
        self.j21 = [np.asarray(m, float).reshape(-1, self.np) for m in j21]
        self.j12 = [(int(r), int(c), np.asarray(b, float)) for (r, c, b) in j12]
        self.r1 = np.ascontiguousarray(r1, float)
        self.r2 = [np.asarray(v, float) for v in r2]
        self.partitions = partitions
        self.sec_off = np.zeros(self.n_cells + 1, np.int32)
        for c in range(self.n_cells):
            self.sec_off[c + 1] = self.sec_off[c] + self.j22[c].shape[0]

    @property
    def n_secondary_total(self) -> int:
        return int(self.sec_off[-1])

    def to_dense_full(self):
        """to_dense_full (condense.cpp:155-180): J over (all primary, all
        secondary) unknowns and -r."""
        n1, n2, np_ = self.n_cells * self.np, self.n_secondary_total, self.np
        so = self.sec_off
        J = np.zeros((n1 + n2, n1 + n2))
        for r in range(self.n_cells):
            for k in range(self.row_ptr[r], self.row_ptr[r + 1]):
                c = self.col_idx[k]
                J[r * np_:(r + 1) * np_, c * np_:(c + 1) * np_] = self.j11_blocks[k]
        for (r, c, b) in self.j12:
            J[r * np_:(r + 1) * np_, n1 + so[c]:n1 + so[c + 1]] += b
        for c in range(self.n_cells):
            if so[c + 1] > so[c]:
                J[n1 + so[c]:n1 + so[c + 1], c * np_:(c + 1) * np_] = self.j21[c]
                J[n1 + so[c]:n1 + so[c + 1], n1 + so[c]:n1 + so[c + 1]] = self.j22[c]
        minus_r = np.concatenate([-self.r1] + [-v for v in self.r2])
        return J, minus_r

    def c_struct(self) -> _GJ:
        """The C ABI view; the packed arrays live on this object."""
        cm = lambda m: np.ascontiguousarray(np.asarray(m, float).T).reshape(-1)  # noqa: E731
        self._p_j11 = np.ascontiguousarray(np.concatenate([cm(b) for b in self.j11_blocks]))
        self._p_j22 = np.ascontiguousarray(np.concatenate([cm(m) for m in self.j22] + [np.zeros(0)]))
        self._p_j21 = np.ascontiguousarray(np.concatenate([cm(m) for m in self.j21] + [np.zeros(0)]))
        self._p_er = np.ascontiguousarray([e[0] for e in self.j12], np.int32)
        self._p_ec = np.ascontiguousarray([e[1] for e in self.j12], np.int32)
        self._p_j12 = np.ascontiguousarray(np.concatenate([cm(e[2]) for e in self.j12] + [np.zeros(0)]))
        self._p_r2 = np.ascontiguousarray(np.concatenate(self.r2 + [np.zeros(0)]))
        p = lambda a: a.ctypes.data  # noqa: E731
        return _GJ(self.n_cells, self.np, p(self.row_ptr), p(self.col_idx), p(self._p_j11), p(self.sec_off),
                   p(self._p_j22), p(self._p_j21), len(self.j12), p(self._p_er), p(self._p_ec), p(self._p_j12),
                   p(self.r1), p(self._p_r2))


def _signed(rng, shape=None):
    m = rng.uniform(0.5, 2.0, size=shape)
    s = rng.integers(0, 2, size=shape)
    return np.where(s == 1, m, -m)


def make_cell_secondary_blocks(vp: VariablePartition, rng):
    """make_cell_secondary_blocks (condense.cpp:318-356): fugacity rows touch their
    aligned unknown's phase counterpart and P, T; phase-constraint rows touch
    every mole fraction of their phase; J22 diagonally dominant."""
    ns, np_ = vp.n_secondary, vp.n_primary
    prim = vp.canonical_labels()
    p_col, t_col = prim.index((PRESSURE, 0)), prim.index((TEMPERATURE, 0))
    j22, j21 = np.zeros((ns, ns)), np.zeros((ns, np_))
    for r in range(ns):
        kind, _ = vp.equations[r]
        if kind == FUGACITY:
            other = _counterpart(vp.secondary[r])
            if other in vp.secondary:
                j22[r, vp.secondary.index(other)] = _signed(rng)
            if other in prim:
                j21[r, prim.index(other)] = _signed(rng)
            j21[r, p_col] = _signed(rng)
            j21[r, t_col] = _signed(rng)
        else:
            phase = VAPOR_FRAC if kind == GAS_CONSTRAINT else OIL_FRAC
            for c in range(ns):
                if c != r and vp.secondary[c][0] == phase:
                    j22[r, c] = _signed(rng)
            for c in range(np_):
                if prim[c][0] == phase:
                    j21[r, c] = _signed(rng)
        j22[r, r] = np.abs(j22[r]).sum() + np.abs(j21[r]).sum() + rng.uniform(0.5, 2.0)
    j12_own = 0.1 * _signed(rng, (np_, ns))
    return j22, j21, j12_own


def make_synthetic_global(states, n_c: int, n_s: int, seed: int, inter_cell_coupling: bool = True) -> GlobalJacobian:
    """make_synthetic_global (condense.cpp:359-421) on a 1-D chain of cells."""
    rng = np.random.default_rng(seed)
    nc = len(states)
    parts = [ordering_for(s, n_c, n_s) for s in states]
    np_ = n_c + n_s + 1
    diag = [_signed(rng, (np_, np_)) for _ in range(nc)]
    blocks = {}
    if inter_cell_coupling:
        for c in range(nc - 1):
            hi, lo = 0.3 * _signed(rng, (np_, np_)), 0.3 * _signed(rng, (np_, np_))
            blocks[(c, c + 1)] = hi
            blocks[(c + 1, c)] = lo
            diag[c][np.diag_indices(np_)] += np.abs(hi).sum(axis=1)
            diag[c + 1][np.diag_indices(np_)] += np.abs(lo).sum(axis=1)
    for c in range(nc):
        d = diag[c]
        for r in range(np_):
            off = np.abs(d[r]).sum() - abs(d[r, r])
            d[r, r] = off + d[r, r] + (1.0 if d[r, r] >= 0.0 else -1.0) * rng.uniform(0.5, 2.0)
        blocks[(c, c)] = d
    keys = sorted(blocks)
    rp = np.zeros(nc + 1, np.int32)
    for (r, _c) in keys:
        rp[r + 1] += 1
    rp = np.cumsum(rp).astype(np.int32)
    ci = np.array([k[1] for k in keys], np.int32)
    j11 = np.stack([blocks[k] for k in keys])
    j22, j21, j12, r2 = [], [], [], []
    for c in range(nc):
        a22, a21, own = make_cell_secondary_blocks(parts[c], rng)
        j22.append(a22)
        j21.append(a21)
        j12.append((c, c, own))
        if inter_cell_coupling and c + 1 < nc:
            j12.append((c, c + 1, 0.05 * _signed(rng, (np_, parts[c + 1].n_secondary))))
        r2.append(rng.uniform(-1.0, 1.0, parts[c].n_secondary))
    r1 = rng.uniform(-1.0, 1.0, nc * np_)
    return GlobalJacobian(nc, np_, rp, ci, j11, j22, j21, j12, r1, r2, parts)


def mixed_states(n: int, seed: int) -> list:
    """A deterministic mix of G / OG / OWG cells (acceptance.cpp: mixed_states)."""
    rng = np.random.default_rng(seed)
    return [STATES[int(k)] for k in rng.integers(0, 3, size=n)]


class PackedGlobalJacobian:
    """A GlobalJacobian already in the C ABI's packed column-major arrays
    (for large systems; see make_synthetic_global_bulk)."""

    def __init__(self, n_cells, np_, row_ptr, col_idx, j11, sec_off, j22, j21, e_row, e_col, j12, r1, r2):
        self.n_cells, self.np = int(n_cells), int(np_)
        a32 = lambda a: np.ascontiguousarray(a, np.int32)  # noqa: E731
        f64 = lambda a: np.ascontiguousarray(a, np.float64)  # noqa: E731
        self.row_ptr, self.col_idx, self.sec_off = a32(row_ptr), a32(col_idx), a32(sec_off)
        self.e_row, self.e_col = a32(e_row), a32(e_col)
        self.j11, self.j22, self.j21, self.j12, self.r1, self.r2 = map(f64, (j11, j22, j21, j12, r1, r2))

    @property
    def n_secondary_total(self) -> int:
        return int(self.sec_off[-1])

    def bytes(self) -> int:
        return sum(a.nbytes for a in (self.row_ptr, self.col_idx, self.sec_off, self.e_row, self.e_col, self.j11,
                                      self.j22, self.j21, self.j12, self.r1, self.r2))

    def c_struct(self) -> _GJ:
        p = lambda a: a.ctypes.data  # noqa: E731
        return _GJ(self.n_cells, self.np, p(self.row_ptr), p(self.col_idx), p(self.j11), p(self.sec_off),
                   p(self.j22), p(self.j21), int(self.e_row.size), p(self.e_row), p(self.e_col), p(self.j12),
                   p(self.r1), p(self.r2))


def _cell_template(vp: VariablePartition):
    """Structural pattern of make_cell_secondary_blocks for one phase state:
    (j22 off-diagonal mask, j21 mask)."""
    ns, np_ = vp.n_secondary, vp.n_primary
    prim = vp.canonical_labels()
    p_col, t_col = prim.index((PRESSURE, 0)), prim.index((TEMPERATURE, 0))
    m22, m21 = np.zeros((ns, ns), bool), np.zeros((ns, np_), bool)
    for r in range(ns):
        kind, _ = vp.equations[r]
        if kind == FUGACITY:
            other = _counterpart(vp.secondary[r])
            if other in vp.secondary:
                m22[r, vp.secondary.index(other)] = True
            if other in prim:
                m21[r, prim.index(other)] = True
            m21[r, p_col] = m21[r, t_col] = True
        else:
            phase = VAPOR_FRAC if kind == GAS_CONSTRAINT else OIL_FRAC
            for c in range(ns):
                if c != r and vp.secondary[c][0] == phase:
                    m22[r, c] = True
            for c in range(np_):
                if prim[c][0] == phase:
                    m21[r, c] = True
    return m22, m21


def make_synthetic_global_bulk(states, n_c: int, n_s: int, seed: int) -> PackedGlobalJacobian:
    """make_synthetic_global's structure (1-D chain with inter-cell coupling),
    vectorised per phase state, packed for the C ABI directly."""
    rng = np.random.default_rng(seed)
    st = np.asarray([STATES.index(s) if isinstance(s, str) else int(s) for s in states], np.int64)
    nc = st.size
    np_ = n_c + n_s + 1
    parts = [ordering_for(s, n_c, n_s) for s in STATES]
    ns_of = np.array([p.n_secondary for p in parts])[st]
    sec_off = np.zeros(nc + 1, np.int64)
    sec_off[1:] = np.cumsum(ns_of)
    # J11: 1-D chain, blocks (c, c-1), (c, c), (c, c+1); column-major blocks
    hi = 0.3 * _signed(rng, (max(nc - 1, 0), np_, np_))
    lo = 0.3 * _signed(rng, (max(nc - 1, 0), np_, np_))
    d = _signed(rng, (nc, np_, np_))
    idx = np.arange(np_)
    d[:-1, idx, idx] += np.abs(hi).sum(axis=2)
    d[1:, idx, idx] += np.abs(lo).sum(axis=2)
    off = np.abs(d).sum(axis=2) - np.abs(d[:, idx, idx])
    dd = d[:, idx, idx]
    d[:, idx, idx] = off + dd + np.where(dd >= 0.0, 1.0, -1.0) * rng.uniform(0.5, 2.0, (nc, np_))
    cnt = np.full(nc, 3)
    cnt[0] -= 1
    cnt[-1] -= 1
    if nc == 1:
        cnt[0] = 1
    row_ptr = np.zeros(nc + 1, np.int64)
    row_ptr[1:] = np.cumsum(cnt)
    nnzb = int(row_ptr[-1])
    col_idx = np.empty(nnzb, np.int64)
    j11 = np.empty((nnzb, np_, np_))
    cells = np.arange(nc)
    first = row_ptr[:-1]
    has_lo = cells > 0
    # positions: lo block (c, c-1) first, then diag, then hi (c, c+1)
    lo_pos = first[has_lo]
    col_idx[lo_pos] = cells[has_lo] - 1
    j11[lo_pos] = lo
    dpos = first + has_lo
    col_idx[dpos] = cells
    j11[dpos] = d
    has_hi = cells < nc - 1
    hi_pos = dpos[has_hi] + 1
    col_idx[hi_pos] = cells[has_hi] + 1
    j11[hi_pos] = hi
    j11 = np.ascontiguousarray(j11.transpose(0, 2, 1)).reshape(-1)
    # per-cell secondary blocks, by state
    n22 = np.zeros(nc + 1, np.int64)
    n22[1:] = np.cumsum(ns_of * ns_of)
    j22 = np.zeros(int(n22[-1]))
    j21 = np.zeros(int(sec_off[-1]) * np_)
    own = np.zeros(int(sec_off[-1]) * np_)
    for s_id, vp in enumerate(parts):
        cs = np.nonzero(st == s_id)[0]
        if cs.size == 0:
            continue
        ns = vp.n_secondary
        m22, m21 = _cell_template(vp)
        a22 = np.where(m22, _signed(rng, (cs.size, ns, ns)), 0.0)
        a21 = np.where(m21, _signed(rng, (cs.size, ns, np_)), 0.0)
        di = np.arange(ns)
        a22[:, di, di] = np.abs(a22).sum(axis=2) + np.abs(a21).sum(axis=2) + rng.uniform(0.5, 2.0, (cs.size, ns))
        pos22 = n22[cs][:, None] + np.arange(ns * ns)[None, :]
        j22[pos22] = a22.transpose(0, 2, 1).reshape(cs.size, -1)
        pos21 = (sec_off[cs] * np_)[:, None] + np.arange(ns * np_)[None, :]
        j21[pos21] = a21.transpose(0, 2, 1).reshape(cs.size, -1)
        o = 0.1 * _signed(rng, (cs.size, np_, ns))
        own[pos21] = o.transpose(0, 2, 1).reshape(cs.size, -1)
    # J12 list: (c, c) own, then (c, c+1) neighbour (np x ns_{c+1})
    e_row = np.repeat(cells, 1 + has_hi)
    e_col = e_row.copy()
    nb_first = np.zeros(nc, np.int64)
    nb_first[1:] = np.cumsum(1 + has_hi)[:-1]
    e_col[nb_first[has_hi] + 1] = cells[has_hi] + 1
    e_ns = ns_of[e_col]
    e_off = np.zeros(e_row.size + 1, np.int64)
    e_off[1:] = np.cumsum(e_ns * np_)
    j12 = np.zeros(int(e_off[-1]))
    own_e = nb_first
    # own blocks: copy from `own` (np x ns_c column-major == the same packing)
    for s_id, vp in enumerate(parts):
        cs = np.nonzero(st == s_id)[0]
        if cs.size == 0:
            continue
        ln = vp.n_secondary * np_
        src = (sec_off[cs] * np_)[:, None] + np.arange(ln)[None, :]
        dst = e_off[own_e[cs]][:, None] + np.arange(ln)[None, :]
        j12[dst] = own[src]
        # neighbour blocks pointing at cells of this state
        nbc = cs[cs > 0]  # column cell of the (c-1, c) neighbour entry
        if nbc.size:
            dst = e_off[nb_first[nbc - 1] + 1][:, None] + np.arange(ln)[None, :]
            j12[dst] = 0.05 * _signed(rng, (nbc.size, ln))
    r2 = rng.uniform(-1.0, 1.0, int(sec_off[-1]))
    r1 = rng.uniform(-1.0, 1.0, nc * np_)
    return PackedGlobalJacobian(nc, np_, row_ptr, col_idx, j11, sec_off, j22, j21, e_row, e_col, j12, r1, r2)
