"""Diagnostics: setup phase breakdown (MPREC_TRACE=1) on one BASELINE config.
python scripts/setup_profile.py CID [method]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("MPREC_TRACE", "1")
from paper_1912_04385_b200 import gen  # noqa: E402
from paper_1912_04385_b200.api import gpu  # noqa: E402

cid = int(sys.argv[1])
method = sys.argv[2] if len(sys.argv) > 2 else gen.CONFIG_METHODS[cid][-1]
api = gpu()
a, b, _ = gen.generate(cid)
t = time.perf_counter()
s = api.system(a).setup(method, b)
print(f"setup {method}: {time.perf_counter() - t:.2f} s", flush=True)
