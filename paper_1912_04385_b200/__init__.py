"""B200-native GMRES / CPR / CPTR3 solve path (arXiv 1912.04385).

The product is the sm_100a library `libmprec_gpu.so` behind the C ABI in
include/mprec_gpu.h; `api` binds it with ctypes for tests and the bench.
"""
from .api import (Api, BlockMatrix, ScalarMatrix, SolveResult, MprecError, DimensionError,  # noqa: F401
                  SingularBlockError, ZeroPivotError, SetupError, ConfigError, CudaError, parse_method,
                  method_name, gpu)
