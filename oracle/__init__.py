"""CPU oracle of the reference solve path -- TEST INFRASTRUCTURE.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
--impl reference) may import this package; it is the checker, never the
thing measured as the product.  See oracle.hpp for what is restated from
where.
"""
import ctypes as _C
import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))
LIB = _os.path.join(_HERE, "liboracle.so")
_api = None


def api():
    """Api (paper_1912_04385_b200.api.Api) bound to liboracle.so with prefix orc_."""
    global _api
    if _api is None:
        from paper_1912_04385_b200.api import Api
        if not _os.path.exists(LIB):
            raise ImportError(f"{LIB} missing: run __graft_entry__.build()")
        _api = Api(LIB, "orc_")
        L = _api.lib
        vp = _C.c_void_p
        for name, args in (("orc_ilu_scalar_factor", [vp, vp]), ("orc_ilu_scalar_apply", [vp, vp, vp]),
                           ("orc_spmv_scalar", [vp, vp, vp]), ("orc_level_sets", [vp, vp])):
            f = getattr(L, name)
            f.restype = _C.c_int
            f.argtypes = args
    return _api


REF_LIB = _os.path.join(_HERE, "_ref", "libmprec_ref.so")
_ref_api = None


def ref_available() -> bool:
    return _os.path.exists(REF_LIB)


def ref_api():
    """Api bound to oracle/_ref/libmprec_ref.so (prefix ref_): the reference's
    own sources compiled against the Eigen-subset shim (oracle/Makefile `ref`)."""
    global _ref_api
    if _ref_api is None:
        from paper_1912_04385_b200.api import Api
        if not ref_available():
            raise ImportError(f"{REF_LIB} missing: run `make -C oracle ref` where /root/reference exists")
        _ref_api = Api(REF_LIB, "ref_")
    return _ref_api
