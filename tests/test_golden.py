"""Committed golden fixtures (tests/golden/make_golden.py).

CPU: the oracle reproduces them exactly on this host (pins the generator and
the oracle across machines -- the fixtures were generated in another
container).  GPU: the sm_100a library matches them (C/F bitwise, scaled
system and ILU digests bitwise, iterations +-1, x within 1e-6)."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
import make_golden as mg  # noqa: E402

GOLD = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_golden.npz"))


def _check(name, r, exact):
    assert str(GOLD[f"{name}/scaled_digest"]) == r["scaled_digest"]
    assert str(GOLD[f"{name}/ilu_digest"]) == r["ilu_digest"]
    for st, lv in enumerate(r["level_sizes"]):
        assert np.array_equal(GOLD[f"{name}/sizes/{st}"], np.array(lv, np.int64))
    for st, levels in enumerate(r["cf"]):
        for l, bits in enumerate(levels):
            assert np.array_equal(GOLD[f"{name}/cf/{st}/{l}"], bits), f"C/F stage {st} level {l}"
    if exact:
        assert int(GOLD[f"{name}/iterations"]) == r["iterations"]
        assert np.array_equal(GOLD[f"{name}/history"], r["history"])
        assert np.array_equal(GOLD[f"{name}/x"], r["x"])
    else:
        assert abs(int(GOLD[f"{name}/iterations"]) - r["iterations"]) <= 1
        x0 = GOLD[f"{name}/x"]
        assert np.linalg.norm(r["x"] - x0) / np.linalg.norm(x0) < 1e-6


@pytest.mark.parametrize("name", list(mg.CASES))
def test_inputs_are_host_independent(name):
    spec = mg.CASES[name][0]
    a, b, _ = mg.system(spec)
    assert str(GOLD[f"{name}/input_digest"]) == mg.digest(a.values) + mg.digest(b)


@pytest.mark.parametrize("name", list(mg.CASES))
def test_oracle_reproduces_golden(orc, name):
    spec, method, amg = mg.CASES[name]
    _check(name, mg.run_case(orc, spec, method, amg), exact=True)


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(mg.CASES))
def test_gpu_matches_golden(gpu, name):
    spec, method, amg = mg.CASES[name]
    _check(name, mg.run_case(gpu, spec, method, amg), exact=False)
