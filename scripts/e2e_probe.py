import ctypes as C, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1912_04385_b200 import gen
from paper_1912_04385_b200.api import gpu, _Result, _ptr
api = gpu()
a, b, xs = gen.generate(5)
for rep in range(2):
    x = np.zeros(a.dim); r2 = _Result()
    t0 = time.perf_counter()
    api.call("solve_system", C.byref(a._c), _ptr(b), 3, 1e-8, 5, _ptr(x), C.byref(r2))
    print(f"rep {rep}: wall {time.perf_counter()-t0:.2f}s setup_s {r2.setup_s:.2f} solve_s {r2.solve_s:.2f}", flush=True)
