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
