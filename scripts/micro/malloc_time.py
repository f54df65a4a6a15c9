import ctypes, time
rt = ctypes.CDLL("libcudart.so.12")
rt.cudaFree(0)
p = ctypes.c_void_p()
ts=[]
ptrs=[]
for i in range(40):
    t=time.perf_counter(); rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(2<<30)); ts.append(time.perf_counter()-t); ptrs.append(p.value)
print("cudaMalloc 2GB ms: first %.2f, mean %.2f, max %.2f" % (ts[0]*1e3, sum(ts)/len(ts)*1e3, max(ts)*1e3))
t=time.perf_counter()
for q in ptrs: rt.cudaFree(ctypes.c_void_p(q))
print("cudaFree 40x2GB total ms %.1f" % ((time.perf_counter()-t)*1e3))
