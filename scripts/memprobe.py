import sys, os
sys.path.insert(0, '/root/repo')
import torch
from paper_1912_04385_b200 import gen
from paper_1912_04385_b200.api import gpu
api = gpu()
a, b, _ = gen.generate(5)
f0, t0 = torch.cuda.mem_get_info()
s = api.system(a).setup("cptr3-amg", b)
f1, _ = torch.cuda.mem_get_info()
r = s.solve(1e-8, 500)
f2, _ = torch.cuda.mem_get_info()
print(f"total {t0/1e9:.1f} GB free: start {f0/1e9:.1f} after setup {f1/1e9:.1f} after 500-it solve {f2/1e9:.1f}")
