"""Profile region = one short GPU solve after an untimed setup + warm-up, for
`ncu --profile-from-start off` (python scripts/profile_solve.py CID max_iter)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 5
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 3
api = gpu()
a, b, _ = gen.generate(cid)
s = api.system(a).setup("cptr3-amg", b)
s.solve(1e-8, 2)  # warm-up
rt = ctypes.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else ctypes.CDLL("libcudart.so")
rt.cudaProfilerStart()
r = s.solve(1e-8, max_iter)
rt.cudaProfilerStop()
print(f"profiled solve: {r.iterations} iterations")
