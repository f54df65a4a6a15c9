"""Synthetic BASELINE.json systems; ctypes over libmprec_gen.so.

Test/bench input infrastructure only (csrc/gen/mprec_gen.h documents the
generator and the builder decisions)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .api import GEN_LIB, BlockMatrix


class GenSpec(C.Structure):
    _fields_ = [("nx", C.c_int), ("ny", C.c_int), ("nb", C.c_int), ("kappa", C.c_double),
                ("perm_sigma", C.c_double), ("band", C.c_int), ("seed", C.c_uint64)]


_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(GEN_LIB):
            raise ImportError(f"{GEN_LIB} missing: run __graft_entry__.build()")
        _lib = C.CDLL(GEN_LIB)
        _lib.mprec_gen_config.argtypes = [C.c_int, C.POINTER(GenSpec)]
        _lib.mprec_gen_nnzb.restype = C.c_int64
        _lib.mprec_gen_nnzb.argtypes = [C.c_int, C.c_int]
        _lib.mprec_gen_pattern.argtypes = [C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        _lib.mprec_gen_fill.argtypes = [C.POINTER(GenSpec), C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int]
    return _lib


CONFIG_METHODS = {1: ["cpr-amg"], 2: ["cpr-amg", "cptr3-amg"], 3: ["cpr-amg", "cptr3-amg"], 4: ["cptr3-amg"],
                  5: ["cptr3-amg"]}


def config_spec(config_id: int) -> GenSpec:
    s = GenSpec()
    if _load().mprec_gen_config(config_id, C.byref(s)) != 0:
        raise ValueError(f"unknown config {config_id}")
    return s


def make_spec(nx, ny, nb, kappa=1.0, perm_sigma=0.0, band=False, seed=1) -> GenSpec:
    return GenSpec(nx, ny, nb, kappa, perm_sigma, int(band), seed)


def generate(spec, nthreads: int = 0):
    """Returns (BlockMatrix A, b = A x*, x*) for a GenSpec or a config id."""
    if isinstance(spec, int):
        spec = config_spec(spec)
    lib = _load()
    nc = spec.nx * spec.ny
    nnzb = int(lib.mprec_gen_nnzb(spec.nx, spec.ny))
    rp = np.zeros(nc + 1, np.int32)
    ci = np.zeros(nnzb, np.int32)
    lib.mprec_gen_pattern(spec.nx, spec.ny, rp.ctypes.data, ci.ctypes.data)
    vals = np.empty(nnzb * spec.nb * spec.nb)
    xs = np.empty(nc * spec.nb)
    b = np.empty(nc * spec.nb)
    if lib.mprec_gen_fill(C.byref(spec), rp.ctypes.data, ci.ctypes.data, vals.ctypes.data, xs.ctypes.data,
                          b.ctypes.data, nthreads) != 0:
        raise ValueError("generator rejected the spec")
    return BlockMatrix(nc, spec.nb, rp, ci, vals), b, xs
