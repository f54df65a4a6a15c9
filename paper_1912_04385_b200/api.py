"""ctypes binding of the C ABI in include/mprec_gpu.h.

The classes mirror the reference's C++ interface for the solve path
(proj/include/mprec/{scaling,stages,amg,ilu0,gmres,harness}.hpp) with the same
names, argument meaning and error classes (proj/include/mprec/errors.hpp), so
tests read like the reference's own tests.  `Api` is generic over the symbol
prefix: the product binds `libmprec_gpu.so` with prefix ``mprec_gpu_``; the
parity tests bind the CPU oracle (`oracle/liboracle.so`, prefix ``orc_``) with
the same wrapper.  This module never loads the oracle itself.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))

# ---- status codes / exceptions (errors.hpp:9-59) ---------------------------
OK, DIMENSION, INDEX, SINGULAR_BLOCK, ZERO_PIVOT, SETUP, CONFIG, INTERNAL, CUDA, IO = range(10)


class MprecError(RuntimeError):
    code = INTERNAL

    def __init__(self, msg: str, payload: int = -1):
        super().__init__(msg)
        self.payload = payload


class DimensionError(MprecError):
    code = DIMENSION


class IndexError_(MprecError):
    code = INDEX


class SingularBlockError(MprecError):
    code = SINGULAR_BLOCK

    @property
    def cell_id(self) -> int:
        return self.payload


class ZeroPivotError(MprecError):
    code = ZERO_PIVOT

    @property
    def row_id(self) -> int:
        return self.payload


class SetupError(MprecError):
    code = SETUP


class ConfigError(MprecError):
    code = CONFIG


class CudaError(MprecError):
    code = CUDA


class IoError(MprecError):
    code = IO


_ERRORS = {c.code: c for c in (DimensionError, IndexError_, SingularBlockError, ZeroPivotError,
                               SetupError, ConfigError, CudaError, IoError)}

# ---- methods (scaling.cpp:5-15) ---------------------------------------------
METHOD_ILU0, METHOD_CPR_AMG, METHOD_CPR_DIRECT, METHOD_CPTR3_AMG, METHOD_CPTR_DIRECT, METHOD_CPTR3_DIRECT = range(6)
_METHODS = {"ilu0": METHOD_ILU0, "cpr-amg": METHOD_CPR_AMG, "cpr-direct": METHOD_CPR_DIRECT,
            "cptr3-amg": METHOD_CPTR3_AMG, "cptr-direct": METHOD_CPTR_DIRECT, "cptr3-direct": METHOD_CPTR3_DIRECT}


def parse_method(name: str) -> int:
    """parse_method (proj/src/scaling.cpp:5-15) for the methods of this path."""
    if name == "cptr-amg":
        raise ConfigError("cptr supports only the -direct sub-solver")
    if name not in _METHODS:
        raise ConfigError(f"unknown method '{name}'")
    return _METHODS[name]


def method_name(m: int) -> str:
    return {v: k for k, v in _METHODS.items()}[m]


# ---- ctypes structs ---------------------------------------------------------
class AmgParams(C.Structure):
    _fields_ = [("strength_threshold", C.c_double), ("max_coarse_size", C.c_int), ("max_levels", C.c_int)]


def amg_params(strength_threshold=0.25, max_coarse_size=1000, max_levels=25) -> AmgParams:
    return AmgParams(strength_threshold, max_coarse_size, max_levels)


class ScalingOptions(C.Structure):
    """ScalingOptions (scaling.hpp:22-30): diag_mode 0 = DiagMode::Block, 1 = Scalar."""
    _fields_ = [("diag_mode", C.c_int), ("second_scaling_from_original", C.c_int)]


DIAG_BLOCK, DIAG_SCALAR = 0, 1


def scaling_options(diag_mode="block", second_scaling_from_original=False) -> ScalingOptions:
    modes = {"block": DIAG_BLOCK, "scalar": DIAG_SCALAR, DIAG_BLOCK: DIAG_BLOCK, DIAG_SCALAR: DIAG_SCALAR}
    if diag_mode not in modes:
        raise ConfigError(f"unknown diag mode {diag_mode!r}")
    return ScalingOptions(modes[diag_mode], int(bool(second_scaling_from_original)))


class _Bsr(C.Structure):
    _fields_ = [("n_cells", C.c_int), ("nb", C.c_int), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p),
                ("values", C.c_void_p)]


class _Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int), ("row_ptr", C.c_void_p), ("col_idx", C.c_void_p), ("values", C.c_void_p)]


class _Result(C.Structure):
    _fields_ = [("iterations", C.c_int), ("converged", C.c_int), ("breakdown", C.c_int), ("attempts", C.c_int),
                ("history_len", C.c_int), ("final_true_residual", C.c_double), ("setup_s", C.c_double),
                ("solve_s", C.c_double), ("total_iterations", C.c_int),
                ("attempt_iterations", C.c_int * 3), ("attempt_converged", C.c_int * 3),
                ("attempt_tol", C.c_double * 3), ("attempt_true_residual", C.c_double * 3)]


@dataclass
class SolveResult:
    """SolveResult (gmres.hpp:28-36) + SolveOutcome timings (harness.hpp:79-83)."""
    x: np.ndarray
    iterations: int
    converged: bool
    breakdown: bool
    attempts: int
    residual_history: np.ndarray
    final_true_residual: float
    setup_time_s: float
    wall_time_s: float
    total_iterations: int = 0
    attempt_iterations: tuple = ()
    attempt_converged: tuple = ()
    attempt_tol: tuple = ()
    attempt_true_residual: tuple = ()


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class BlockMatrix:
    """Uniform-layout BlockMatrix (block_matrix.hpp:50-101): BSR with column-major
    nb x nb blocks in (s..., P, T) intra-cell order."""

    def __init__(self, n_cells: int, nb: int, row_ptr, col_idx, values):
        self.n_cells, self.nb = int(n_cells), int(nb)
        self.row_ptr, self.col_idx = _i32(row_ptr), _i32(col_idx)
        self.values = _f64(values).reshape(-1)
        if self.values.size != self.col_idx.size * nb * nb:
            raise DimensionError("values size does not match nnzb * nb * nb")
        self._c = _Bsr(self.n_cells, self.nb, _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.values))

    @property
    def dim(self) -> int:
        return self.n_cells * self.nb

    @property
    def nnzb(self) -> int:
        return int(self.col_idx.size)

    def blocks(self) -> np.ndarray:
        """(nnzb, nb, nb) row-major view (block[k][r][c])."""
        return self.values.reshape(-1, self.nb, self.nb).transpose(0, 2, 1)

    def to_dense(self) -> np.ndarray:
        nb = self.nb
        d = np.zeros((self.dim, self.dim))
        b = self.blocks()
        for c in range(self.n_cells):
            for k in range(self.row_ptr[c], self.row_ptr[c + 1]):
                j = self.col_idx[k]
                d[c * nb:(c + 1) * nb, j * nb:(j + 1) * nb] = b[k]
        return d

    @staticmethod
    def from_dense_blocks(n_cells: int, nb: int, blocks: dict) -> "BlockMatrix":
        """BlockMatrix::assemble (block_matrix.cpp:32-69): {(row,col): (nb,nb) array};
        duplicates must be merged by the caller; a zero diagonal block is added
        where none is given."""
        bl = dict(blocks)
        for c in range(n_cells):
            bl.setdefault((c, c), np.zeros((nb, nb)))
        keys = sorted(bl)
        rp = np.zeros(n_cells + 1, np.int32)
        ci = np.array([k[1] for k in keys], np.int32)
        vals = np.concatenate([np.asarray(bl[k], float).T.reshape(-1) for k in keys])
        for (r, _c) in keys:
            rp[r + 1] += 1
        rp = np.cumsum(rp).astype(np.int32)
        return BlockMatrix(n_cells, nb, rp, ci, vals)


class ScalarMatrix:
    """Canonical CSR (scalar_matrix.hpp:20-62)."""

    def __init__(self, n: int, row_ptr, col_idx, values):
        self.n = int(n)
        self.row_ptr, self.col_idx, self.values = _i32(row_ptr), _i32(col_idx), _f64(values)
        self._c = _Csr(self.n, _ptr(self.row_ptr), _ptr(self.col_idx), _ptr(self.values))

    @staticmethod
    def from_triplets(n: int, triplets) -> "ScalarMatrix":
        """from_triplets (scalar_matrix.cpp:8-35): sort, sum duplicates."""
        acc: dict = {}
        for (i, j, v) in triplets:
            acc[(i, j)] = acc.get((i, j), 0.0) + v
        keys = sorted(acc)
        rp = np.zeros(n + 1, np.int64)
        for (i, _j) in keys:
            rp[i + 1] += 1
        return ScalarMatrix(n, np.cumsum(rp), [k[1] for k in keys], [acc[k] for k in keys])

    def to_dense(self) -> np.ndarray:
        d = np.zeros((self.n, self.n))
        for i in range(self.n):
            for k in range(self.row_ptr[i], self.row_ptr[i + 1]):
                d[i, self.col_idx[k]] = self.values[k]
        return d

    def as_block(self) -> BlockMatrix:
        return BlockMatrix(self.n, 1, self.row_ptr, self.col_idx, self.values)


class Api:
    """Binding of one implementation of the C ABI (GPU library or CPU oracle)."""

    def __init__(self, lib_path: str, prefix: str):
        self.lib = C.CDLL(lib_path)
        self.prefix = prefix
        self.path = lib_path
        L, p = self.lib, prefix
        vp, ip, dp, i64p = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int64)
        sig = {
            "last_error": (C.c_char_p, []),
            "error_payload": (C.c_int, []),
            "create": (C.c_int, [vp, C.POINTER(vp)]),
            "setup": (C.c_int, [vp, C.c_int, vp, vp]),
            "apply": (C.c_int, [vp, vp, vp]),
            "apply_stage": (C.c_int, [vp, C.c_int, vp, vp]),
            "spmv": (C.c_int, [vp, C.c_int, vp, vp]),
            "solve": (C.c_int, [vp, C.c_double, C.c_int, vp, vp, vp, C.c_int]),
            "get_scaled": (C.c_int, [vp, vp, vp]),
            "get_ilu": (C.c_int, [vp, vp]),
            "n_stages": (C.c_int, [vp, ip]),
            "stage_amg": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
            "destroy": (None, [vp]),
            "amg_create": (C.c_int, [vp, vp, C.POINTER(vp)]),
            "amg_apply": (C.c_int, [vp, vp, vp]),
            "amg_n_levels": (C.c_int, [vp, ip]),
            "amg_level_info": (C.c_int, [vp, C.c_int, ip, ip, ip]),
            "amg_get_csr": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp]),
            "amg_get_cf": (C.c_int, [vp, C.c_int, vp]),
            "amg_destroy": (None, [vp]),
            "ilu_create": (C.c_int, [vp, C.POINTER(vp)]),
            "ilu_apply": (C.c_int, [vp, vp, vp]),
            "ilu_get": (C.c_int, [vp, vp]),
            "ilu_destroy": (None, [vp]),
            "gmres": (C.c_int, [vp, vp, C.c_int, vp, C.c_double, C.c_int, vp, vp, vp, C.c_int]),
        }
        optional = {
            "setup_opts": (C.c_int, [vp, C.c_int, vp, vp, vp]),
            "scaling_record": (C.c_int, [vp, C.c_char_p, C.c_int]),
            "get_levelsets": (C.c_int, [vp, C.c_int, vp, ip]),
            "amg_get_levelsets": (C.c_int, [vp, C.c_int, C.c_int, vp, ip]),
            "solve_dev": (C.c_int, [vp, C.c_double, C.c_int, vp, vp]),
            "last_history": (C.c_int, [vp, vp, C.c_int, vp]),
            "solve_system": (C.c_int, [vp, vp, C.c_int, C.c_double, C.c_int, vp, vp]),
            "device_info": (C.c_int, [ip, ip, ip, i64p]),
            "profile": (C.c_int, [vp, C.c_int]),
            "kernel_stats": (C.c_int, [vp, C.c_int, dp, i64p, dp]),
            "reset_stats": (C.c_int, [vp]),
            "launch_count": (C.c_int, [vp, i64p]),
            "stream": (C.c_int, [vp, C.POINTER(vp)]),
            "ingest": (C.c_int, [C.c_char_p, C.c_char_p, C.c_char_p, C.POINTER(vp)]),
            "get_shape": (C.c_int, [vp, ip, ip, ip]),
            "get_matrix": (C.c_int, [vp, vp, vp, vp, vp]),
            "write_system": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_char_p]),
            "condense": (C.c_int, [vp, C.POINTER(vp)]),
            "condensed_shape": (C.c_int, [vp, ip, ip, ip, ip]),
            "condensed_get": (C.c_int, [vp, vp, vp, vp, vp]),
            "condensed_system": (C.c_int, [vp, C.POINTER(vp)]),
            "back_substitute": (C.c_int, [vp, vp, vp]),
            "condensed_destroy": (None, [vp]),
        }
        self.fn = {}
        for name, (res, args) in list(sig.items()) + list(optional.items()):
            try:
                f = getattr(L, p + name)
            except AttributeError:
                if name in sig:
                    raise
                continue
            f.restype = res
            f.argtypes = args
            self.fn[name] = f

    def has(self, name: str) -> bool:
        return name in self.fn

    def check(self, status: int) -> None:
        if status == OK:
            return
        msg = self.fn["last_error"]().decode(errors="replace")
        payload = self.fn["error_payload"]()
        raise _ERRORS.get(status, MprecError)(msg, payload)

    def call(self, name: str, *args) -> None:
        self.check(self.fn[name](*args))

    # ---- factories mirroring the reference API ----
    def system(self, a: BlockMatrix) -> "System":
        return System(self, a)

    def amg(self, a: ScalarMatrix, **params) -> "AMGHierarchy":
        return AMGHierarchy(self, a, amg_params(**params) if params else None)

    def ilu0(self, a) -> "ILU0Factor":
        return ILU0Factor(self, a.as_block() if isinstance(a, ScalarMatrix) else a)

    def ingest(self, matrix_path: str, layout_path: str, rhs_path: str) -> "System":
        """ingest_external (harness.cpp:153-188): Matrix Market + layout + rhs."""
        h = C.c_void_p()
        self.call("ingest", matrix_path.encode(), layout_path.encode(), rhs_path.encode(), C.byref(h))
        nc, nb, nnzb = C.c_int(), C.c_int(), C.c_int()
        self.call("get_shape", h, C.byref(nc), C.byref(nb), C.byref(nnzb))
        rp = np.zeros(nc.value + 1, np.int32)
        ci = np.zeros(nnzb.value, np.int32)
        v = np.zeros(nnzb.value * nb.value * nb.value)
        b = np.zeros(nc.value * nb.value)
        self.call("get_matrix", h, _ptr(rp), _ptr(ci), _ptr(v), _ptr(b))
        sysm = System.__new__(System)
        sysm.api, sysm.a, sysm.h, sysm.method, sysm.b = self, BlockMatrix(nc.value, nb.value, rp, ci, v), h, None, b
        return sysm

    def condense(self, j) -> "ReducedSystem":
        """condense (condense.cpp:206-241) of a condense.GlobalJacobian."""
        gj = j.c_struct()
        h = C.c_void_p()
        self.call("condense", C.byref(gj), C.byref(h))
        return ReducedSystem(self, h)

    def gmres(self, a, b, prec=None, tol=1e-8, max_iter=500) -> SolveResult:
        """gmres (gmres.cpp:8-106); a: BlockMatrix or ScalarMatrix; prec: None
        (identity), AMGHierarchy or ILU0Factor of the same Api."""
        a = a.as_block() if isinstance(a, ScalarMatrix) else a
        b = _f64(b)
        kind, h = 0, None
        if isinstance(prec, AMGHierarchy):
            kind, h = 1, prec.h
        elif isinstance(prec, ILU0Factor):
            kind, h = 2, prec.h
        elif prec is not None:
            raise ConfigError("unsupported preconditioner")
        x = np.zeros(a.dim)
        res = _Result()
        hist = np.zeros(max(min(max_iter, a.dim), 0) + 2)
        self.call("gmres", C.byref(a._c), _ptr(b), kind, h, tol, max_iter, _ptr(x), C.byref(res), _ptr(hist),
                  hist.size)
        return _result(x, res, hist)


def _result(x, res: _Result, hist) -> SolveResult:
    return SolveResult(x=x, iterations=res.iterations, converged=bool(res.converged),
                       breakdown=bool(res.breakdown), attempts=res.attempts,
                       residual_history=np.array(hist[:res.history_len]),
                       final_true_residual=res.final_true_residual, setup_time_s=res.setup_s,
                       wall_time_s=res.solve_s, total_iterations=res.total_iterations,
                       attempt_iterations=tuple(res.attempt_iterations[:max(res.attempts, 0)]),
                       attempt_converged=tuple(bool(c) for c in res.attempt_converged[:max(res.attempts, 0)]),
                       attempt_tol=tuple(res.attempt_tol[:max(res.attempts, 0)]),
                       attempt_true_residual=tuple(res.attempt_true_residual[:max(res.attempts, 0)]))


class System:
    """One system on one implementation: left_scale + build_preconditioner
    (setup), StagePreconditioner::apply, solve_system."""

    def __init__(self, api: Api, a: BlockMatrix):
        self.api, self.a = api, a
        h = C.c_void_p()
        api.call("create", C.byref(a._c), C.byref(h))
        self.h = h
        self.method = None

    def close(self):
        if self.h:
            self.api.fn["destroy"](self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def setup(self, method, b=None, diag_mode="block", second_scaling_from_original=False, **amg) -> "System":
        """left_scale(A, b, method, ScalingOptions{diag_mode, second_scaling_from_original})
        + build_preconditioner(scaled, method, AMGParams{**amg}) (scaling.hpp:65-66, stages.hpp:85-86)."""
        m = parse_method(method) if isinstance(method, str) else int(method)
        if b is None:  # rhs held by the handle (ingested system)
            b = self.b
        self.b = _f64(b)
        if self.b.size != self.a.dim:
            raise DimensionError("rhs length mismatch")
        p = amg_params(**amg) if amg else None
        so = scaling_options(diag_mode, second_scaling_from_original)
        if self.api.has("setup_opts"):
            self.api.call("setup_opts", self.h, m, C.byref(p) if p is not None else None, C.byref(so), _ptr(self.b))
        else:
            if so.diag_mode != DIAG_BLOCK or so.second_scaling_from_original:
                raise ConfigError("this implementation has no ScalingOptions entry point")
            self.api.call("setup", self.h, m, C.byref(p) if p is not None else None, _ptr(self.b))
        self.method = m
        return self

    def scaling_record(self) -> str:
        """SolveOutcome::scaling_record (harness.cpp:197-201): the applied D factors, in order."""
        buf = C.create_string_buffer(256)
        self.api.call("scaling_record", self.h, buf, len(buf))
        return buf.value.decode()

    def write(self, matrix_path: str, layout_path: str, rhs_path: str) -> None:
        """write_block_matrix + write_vector (matrix_io.cpp:93-114); GPU library only."""
        self.api.call("write_system", self.h, matrix_path.encode(), layout_path.encode(), rhs_path.encode())

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        z = np.zeros(self.a.dim)
        self.api.call("apply", self.h, _ptr(r), _ptr(z))
        return z

    def apply_stage(self, i: int, r) -> np.ndarray:
        r = _f64(r)
        z = np.zeros(self.a.dim)
        self.api.call("apply_stage", self.h, i, _ptr(r), _ptr(z))
        return z

    def spmv(self, x, which: int = 0) -> np.ndarray:
        x = _f64(x)
        y = np.zeros(self.a.dim)
        self.api.call("spmv", self.h, which, _ptr(x), _ptr(y))
        return y

    def solve(self, tol=1e-8, max_iter=500) -> SolveResult:
        x = np.zeros(self.a.dim)
        res = _Result()
        hist = np.zeros(max(min(max_iter, self.a.dim), 0) + 2)
        self.api.call("solve", self.h, tol, max_iter, _ptr(x), C.byref(res), _ptr(hist), hist.size)
        return _result(x, res, hist)

    def scaled(self):
        """(a_bar values, b_bar) of the ScaledSystem (scaling.hpp:36-46)."""
        av = np.zeros(self.a.nnzb * self.a.nb * self.a.nb)
        bb = np.zeros(self.a.dim)
        self.api.call("get_scaled", self.h, _ptr(av), _ptr(bb))
        return av, bb

    def ilu_values(self) -> np.ndarray:
        v = np.zeros(self.a.nnzb * self.a.nb * self.a.nb)
        self.api.call("get_ilu", self.h, _ptr(v))
        return v

    def levelsets(self, direction: int = 1):
        """(levels per cell, depth) of the block-row DAG the ILU(0) sweeps are
        scheduled on; direction +1 forward, -1 backward."""
        out = np.zeros(self.a.n_cells, np.int32)
        nl = C.c_int()
        self.api.call("get_levelsets", self.h, int(direction), _ptr(out), C.byref(nl))
        return out, nl.value

    def n_stages(self) -> int:
        n = C.c_int()
        self.api.call("n_stages", self.h, C.byref(n))
        return n.value

    def stage_amg(self, i: int) -> "AMGHierarchy":
        h = C.c_void_p()
        self.api.call("stage_amg", self.h, i, C.byref(h))
        return AMGHierarchy._view(self.api, h, owner=self)


class AMGHierarchy:
    """AMGHierarchy::setup/apply (amg.hpp:21-49)."""

    def __init__(self, api: Api, a: ScalarMatrix, params: AmgParams | None):
        self.api, self.a, self._owner, self._owned = api, a, None, True
        h = C.c_void_p()
        api.call("amg_create", C.byref(a._c), C.byref(params) if params is not None else None, C.byref(h))
        self.h = h

    @classmethod
    def _view(cls, api, h, owner):
        o = cls.__new__(cls)
        o.api, o.a, o.h, o._owner, o._owned = api, None, h, owner, False
        return o

    def __del__(self):
        try:
            if self._owned and self.h:
                self.api.fn["amg_destroy"](self.h)
                self.h = None
        except Exception:
            pass

    @property
    def n_levels(self) -> int:
        n = C.c_int()
        self.api.call("amg_n_levels", self.h, C.byref(n))
        return n.value

    def level_info(self, l: int):
        n, na, npp = C.c_int(), C.c_int(), C.c_int()
        self.api.call("amg_level_info", self.h, l, C.byref(n), C.byref(na), C.byref(npp))
        return n.value, na.value, npp.value

    def level_csr(self, l: int, which: int = 0):
        """(row_ptr, col_idx, values) of A_l (0), P_l (1) or R_l (2)."""
        n, na, npp = self.level_info(l)
        if which == 0:
            rows, nnz = n, na
        else:
            nf, _, _ = self.level_info(l - 1)
            rows, nnz = (nf, npp) if which == 1 else (n, npp)
        rp = np.zeros(rows + 1, np.int32)
        ci = np.zeros(nnz, np.int32)
        v = np.zeros(nnz)
        self.api.call("amg_get_csr", self.h, l, which, _ptr(rp), _ptr(ci), _ptr(v))
        return rp, ci, v

    def cf(self, l: int) -> np.ndarray:
        n, _, _ = self.level_info(l)
        out = np.zeros(n, np.int8)
        self.api.call("amg_get_cf", self.h, l, _ptr(out))
        return out

    def levelsets(self, l: int, direction: int = 1):
        """(levels per row, depth) of level l's Gauss-Seidel sweep DAG."""
        n, _, _ = self.level_info(l)
        out = np.zeros(n, np.int32)
        nl = C.c_int()
        self.api.call("amg_get_levelsets", self.h, l, int(direction), _ptr(out), C.byref(nl))
        return out, nl.value

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        n, _, _ = self.level_info(0)
        x = np.zeros(n)
        self.api.call("amg_apply", self.h, _ptr(r), _ptr(x))
        return x


class ILU0Factor:
    """ILU0Factor::factor/apply (ilu0.hpp:9-24) on a BSR (nb = 1: scalar)."""

    def __init__(self, api: Api, a: BlockMatrix):
        self.api, self.a = api, a
        h = C.c_void_p()
        api.call("ilu_create", C.byref(a._c), C.byref(h))
        self.h = h

    def __del__(self):
        try:
            if self.h:
                self.api.fn["ilu_destroy"](self.h)
                self.h = None
        except Exception:
            pass

    def apply(self, r) -> np.ndarray:
        r = _f64(r)
        y = np.zeros(self.a.dim)
        self.api.call("ilu_apply", self.h, _ptr(r), _ptr(y))
        return y

    def factors(self) -> np.ndarray:
        v = np.zeros_like(self.a.values)
        self.api.call("ilu_get", self.h, _ptr(v))
        return v


# ---- the product library ----------------------------------------------------
# MPREC_LIB=checked: the bounds-checked build (tests/test_checked.py)
GPU_LIB = os.path.join(_HERE, "libmprec_gpu_checked.so" if os.environ.get("MPREC_LIB") == "checked"
                       else "libmprec_gpu.so")
GEN_LIB = os.path.join(_HERE, "libmprec_gen.so")
_gpu_api = None


def gpu() -> Api:
    """The B200 library.  Fails loudly when it is not built: there is no CPU
    fallback on the product path."""
    global _gpu_api
    if _gpu_api is None:
        if not os.path.exists(GPU_LIB):
            raise ImportError(f"{GPU_LIB} missing: run __graft_entry__.build() (no CPU fallback exists)")
        _gpu_api = Api(GPU_LIB, "mprec_gpu_")
    return _gpu_api


class ReducedSystem:
    """ReducedSystem (condense.hpp:83-90): A = J11 - J12 J22^-1 J21,
    b = -r1 + J12 J22^-1 r2, with the J22 factors kept for back_substitute."""

    def __init__(self, api: Api, h):
        self.api, self.h = api, h
        nc, np_, nnzb, n2 = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        api.call("condensed_shape", h, C.byref(nc), C.byref(np_), C.byref(nnzb), C.byref(n2))
        self.n_cells, self.np, self.n_secondary = nc.value, np_.value, n2.value
        rp = np.zeros(nc.value + 1, np.int32)
        ci = np.zeros(nnzb.value, np.int32)
        v = np.zeros(nnzb.value * np_.value * np_.value)
        self.b = np.zeros(nc.value * np_.value)
        api.call("condensed_get", h, _ptr(rp), _ptr(ci), _ptr(v), _ptr(self.b))
        self.a = BlockMatrix(nc.value, np_.value, rp, ci, v)

    def back_substitute(self, d1) -> np.ndarray:
        """back_substitute (condense.cpp:243-258): d2 = J22^-1 (-r2 - J21 d1)."""
        d1 = _f64(d1)
        if d1.size != self.n_cells * self.np:
            raise DimensionError("primary update dimension mismatch")
        d2 = np.zeros(max(self.n_secondary, 1))
        self.api.call("back_substitute", self.h, _ptr(d1), _ptr(d2))
        return d2[: self.n_secondary]

    def system(self) -> "System":
        """A solver System on the reduced A (device to device); its rhs is b."""
        h = C.c_void_p()
        self.api.call("condensed_system", self.h, C.byref(h))
        sysm = System.__new__(System)
        sysm.api, sysm.a, sysm.h, sysm.method, sysm.b = self.api, self.a, h, None, self.b.copy()
        return sysm

    def __del__(self):
        try:
            if self.h:
                self.api.fn["condensed_destroy"](self.h)
                self.h = None
        except Exception:
            pass
