"""Full-size parity of BASELINE configs 4 and 5 (north_star: "matches the CPU
oracle on every config") against the committed oracle records
tests/golden/big_c{4,5}.npz (tests/golden/make_big_golden.py; the oracle itself
is pinned to the reference's own execution by tests/test_ref_pin.py).

  * setup: sha256 digests of the scaled system, the ILU(0) factors and every AMG
    level's C/F splitting, A_l, P_l and R_l -- bitwise;
  * the preconditioner and every stage applied to a seeded r -- 1e-10 relative
    on a strided sample;
  * solve_system (harness.cpp:190-219): c4 takes all three tolerance-tightening
    attempts (harness.cpp:209-217).  These reaction-band systems are so
    ill-conditioned that the oracle's own iteration counts move under a 1e-15
    perturbation of b, so the GPU is held to the oracle's rounding band
    (tests/ensemble.py): iterations per attempt within [min - 1, max + 1] of
    the recorded ensemble, the history within its spread, the same verdicts.
    c5: the first 40 GMRES iterations (the bench runs 500).
"""
import os

import numpy as np
import pytest

from tests.bigcase import run_case
from tests.ensemble import check_history

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _golden(cid):
    path = os.path.join(GOLDEN, f"big_c{cid}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_big_golden.py {cid}")
    z = np.load(path, allow_pickle=False)
    return {k: z[k] for k in z.files}


def _rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _ensemble(go):
    npert = len([k for k in go if k.endswith("_history") and k.startswith("pert")])
    hists = [go["history"]] + [go[f"pert{s}_history"] for s in range(npert)]
    its = [go["attempt_iterations"]] + [go[f"pert{s}_attempt_iterations"] for s in range(npert)]
    return hists, its


def _check(gpu, cid, iters):
    go = _golden(cid)
    gg = run_case(gpu, cid, iters, apply_sample=True, log=lambda m: print(f"gpu c{cid}: {m}"))
    assert str(gg["input"]) == str(go["input"]), "generator output differs from the golden record's"
    # setup: bitwise
    keys = sorted(k for k in go if k in ("scaled", "ilu") or k.startswith("s") and "/" in k)
    assert keys, "golden record has no setup digests"
    bad = [k for k in keys if not np.array_equal(np.asarray(gg.get(k)), np.asarray(go[k]))]
    assert not bad, f"setup differs from the oracle at {bad[:6]}"
    # applications: 1e-10 relative
    assert _rel(gg["apply_sample"], go["apply_sample"]) < 1e-10
    st = 0
    while f"stage{st}_sample" in go:
        assert _rel(gg[f"stage{st}_sample"], go[f"stage{st}_sample"]) < 1e-10, f"stage {st}"
        st += 1
    # solve: the oracle's rounding band
    hists, its = _ensemble(go)
    assert int(gg["attempts"]) == int(go["attempts"])
    assert bool(gg["converged"]) == bool(go["converged"])
    its = np.array([i for i in its if len(i) == len(go["attempt_iterations"])])
    lo, hi = its.min(axis=0), its.max(axis=0)
    for q, ig in enumerate(gg["attempt_iterations"]):
        assert lo[q] - 1 <= ig <= hi[q] + 1, (gg["attempt_iterations"], go["attempt_iterations"], lo, hi)
    tol = 1e-8
    for tg, to in zip(gg["attempt_true_residual"], go["attempt_true_residual"]):
        assert (tg <= tol) == (to <= tol)
    worst = check_history(gg["history"], hists)
    print(f"c{cid}: gpu attempts {list(gg['attempt_iterations'])} oracle {list(go['attempt_iterations'])} "
          f"band {list(lo)}..{list(hi)}; history dev/bound max {worst:.2e}; "
          f"true residual gpu {float(gg['final_true_residual']):.3e} oracle {float(go['final_true_residual']):.3e}")
    return gg, go


def test_c4_solve_system_full(gpu):
    """Config 4 (500x500, nb 8, reaction band, cptr3-amg): the whole solve_system,
    three attempts."""
    gg, go = _check(gpu, 4, 500)
    assert int(go["attempts"]) == 3
    npert = len([k for k in go if k.startswith("pert") and k.endswith("_final_true_residual")])
    finals = [float(go["final_true_residual"])] + [float(go[f"pert{s}_final_true_residual"]) for s in range(npert)]
    ft = float(gg["final_true_residual"])
    assert min(finals) / 10 <= ft <= max(finals) * 10, (ft, finals)


def test_c5_setup_and_first_iterations(gpu):
    """Config 5 (2000x2000, nb 8, 10 GB of blocks): setup bitwise, applications at
    1e-10, the first 40 iterations inside the oracle's band."""
    _check(gpu, 5, 40)


@pytest.mark.parametrize("cid", [4, 5])
def test_levelsets_c4_c5(gpu, cid):
    """north_star "level sets bit-exact" at full size: the level sets of every
    sequential sweep the device schedules (ILU(0) block DAG, Gauss-Seidel on every
    smoothed level of both hierarchies, both directions) equal the oracle's
    (tests/golden/levelsets_c45.npz; c5 level 0: 3,999 levels)."""
    from paper_1912_04385_b200 import gen
    from tests.bigcase import levelset_digests
    path = os.path.join(GOLDEN, "levelsets_c45.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_levelset_golden.py")
    z = np.load(path)
    want = {k.split("/", 1)[1]: str(z[k]) for k in z.files if k.startswith(f"c{cid}/")}
    a, b, _ = gen.generate(cid)
    s = gpu.system(a)
    a.values = None
    s.setup(gen.CONFIG_METHODS[cid][-1], b)
    got = levelset_digests(s)
    assert set(got) == set(want)
    bad = [k for k in want if got[k] != want[k]]
    assert not bad, bad
    if cid == 5:
        assert want["ilu/d1"].endswith(":3999")
