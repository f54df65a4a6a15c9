"""Diagnostics: distribution of solve_system attempt iterations under 1e-15
perturbations of b (tests/ensemble.py) on one RETRY_SPECS system.

    python scripts/retry_dist.py IMPL NAME [runs]      IMPL = gpu | oracle
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.ensemble import perturbed  # noqa: E402
from tests.systems import retry_system  # noqa: E402

impl, name = sys.argv[1], sys.argv[2]
runs = int(sys.argv[3]) if len(sys.argv) > 3 else 20
if impl == "gpu":
    from paper_1912_04385_b200.api import gpu
    api = gpu()
else:
    import oracle
    api = oracle.api()
a, b, xs, m = retry_system(name)
its = []
for s in [None] + list(range(runs)):
    bb = b if s is None else perturbed(b, s)
    r = api.system(a).setup(m, bb, max_coarse_size=40).solve()
    its.append(r.attempt_iterations)
its = np.array(its)
print(f"{impl} {name}: unperturbed {tuple(its[0])}; {runs} perturbed: min {its[1:].min(0)} max {its[1:].max(0)} "
      f"mean {its[1:].mean(0).round(1)}")
