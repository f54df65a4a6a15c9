"""Sweep harness (harness.cpp:13-421): ports of proj/tests/test_harness.cpp.

CPU tests drive the harness through the oracle's C ABI; the GPU test runs the
same sweep through the product library and compares row by row.
"""
import os

import numpy as np
import pytest

from paper_1912_04385_b200 import api as A
from paper_1912_04385_b200 import sweep as S

CONFIG = """
# sweep with two scenarios
[sweep]
seed = 7
output = out_dir

[scenario]
name = low
nx = 6
ny = 6
n_c = 3
pe = 0.01
method = cpr-direct

[scenario]
name = high ; trailing comment
nx = 6
ny = 6
n_c = 3
pe = 100
method = cptr3-direct
tol = 1e-9
max_iter = 200
"""


def test_config_parsing():
    cfg = S.parse_config_stream(CONFIG, "inline")
    assert cfg.seed == 7 and cfg.output_dir == "out_dir"
    assert len(cfg.scenarios) == 2
    s0, s1 = cfg.scenarios
    assert (s0.name, s0.nx, s0.n_c, s0.pe, s0.method, s0.tol) == ("low", 6, 3, 0.01, "cpr-direct", 1e-8)
    assert (s1.method, s1.tol, s1.max_iter) == ("cptr3-direct", 1e-9, 200)


@pytest.mark.parametrize("text", [
    "[scenario]\nname = a\nbogus = 1\n",
    "[sweep]\nseed = 1\n",
    "[scenario]\nmethod = cg\n",
    "[scenario]\nmethod = cptr-amg\n",
    "[scenario]\ntol = 2.0\n",
    "[scenario]\nmax_iter = 0\n",
    "seed = 1\n",
    "[mystery]\n",
    "[scenario\n",
    "[scenario]\nnx = 2.5\n",
    "[scenario]\nnx = ten\n",
])
def test_config_rejects_malformed(text):
    with pytest.raises(A.ConfigError):
        S.parse_config_stream(text, "inline")


def test_parse_config_missing_file():
    with pytest.raises(A.ConfigError):
        S.parse_config("/nonexistent/sweep.ini")


def test_cv_population():
    assert S.compute_cv([10.0, 10.0, 10.0]) == 0.0
    assert abs(S.compute_cv([5.0, 10.0, 15.0]) - 40.8248) < 1e-4 * 40.8248
    with pytest.raises(A.ConfigError):
        S.compute_cv([])
    with pytest.raises(A.ConfigError):
        S.compute_cv([1.0, -1.0])


def test_cv_sample_published_counts():
    """criterion 10 (acceptance.cpp:395-406): 41.6 % and 12.8 %."""
    assert abs(S.compute_cv_sample([42.0, 20.0, 50.0]) - 41.6) < 0.5
    assert abs(S.compute_cv_sample([15.0, 12.0, 15.0]) - 12.8) < 0.5
    with pytest.raises(A.ConfigError):
        S.compute_cv_sample([3.0])


def test_kappa_for_peclet():
    assert S.kappa_for_peclet(1.0) == pytest.approx(4.32 * 3.1 * 1.42 / 0.35)
    with pytest.raises(A.ConfigError):
        S.kappa_for_peclet(0.0)


def _identity_system(api):
    n_cells, nb = 4, 4
    blocks = {(c, c): np.eye(nb) for c in range(n_cells)}
    return api.system(A.BlockMatrix.from_dense_blocks(n_cells, nb, blocks)), 1.0 + np.arange(16.0)


@pytest.mark.parametrize("method", ["ilu0", "cpr-direct", "cptr-direct", "cptr3-direct"])
def test_identity_one_iteration(orc, method):
    s, b = _identity_system(orc)
    r = s.setup(method, b).solve()
    assert r.converged and r.iterations == 1 and r.final_true_residual < 1e-12


def _pe_config():
    cfg = S.ExperimentConfig(seed=7)
    for method in ("cpr-direct", "cptr3-direct"):
        for pe in (1e-2, 1.0, 1e2):
            cfg.scenarios.append(S.Scenario(name=f"{method}@{pe}", nx=6, ny=6, n_c=3, pe=pe, method=method))
    return cfg


def _check_pe_report(rep):
    assert len(rep.rows) == 6
    for row in rep.rows:
        assert row.error == "" and row.converged
        assert row.grid == "6x6" and row.matrix_dim == 6 * 6 * 5
        assert row.iterations > 0 and row.final_true_resid < 1e-7
    assert [c.method for c in rep.cv] == ["cpr-direct", "cptr3-direct"]
    assert all(c.cv_percent >= 0.0 for c in rep.cv)
    # the stronger method varies less across the Peclet axis (test_harness.cpp:137-138)
    assert rep.cv[1].cv_percent <= rep.cv[0].cv_percent


def test_sweep_rows_and_cv(orc):
    _check_pe_report(S.run_sweep(_pe_config(), orc))


def test_failing_scenario_is_a_row_error(orc):
    cfg = S.ExperimentConfig(scenarios=[S.Scenario(name="missing", basename="no_such_basename")])
    rep = S.run_sweep(cfg, orc)
    assert len(rep.rows) == 1 and rep.rows[0].error != "" and rep.cv == []


def test_csv_round_trip_and_strip(tmp_path):
    rep = S.IterationReport([S.ReportRow("s1", "cpr-amg", "40x40", 0.01, 22400, 123, 70, True, 3.25e-9, 0.5, 1.5, "")],
                            [S.CvRow("cpr-amg", "40x40", 63.0)])
    base = str(tmp_path / "rt_test")
    S.emit_report(rep, "csv", base)
    back = S.parse_report_csv(base)
    assert len(back.rows) == 1
    r = back.rows[0]
    assert (r.scenario, r.iterations, r.final_true_resid, r.setup_time) == ("s1", 70, 3.25e-9, 0.5)
    assert len(back.cv) == 1 and back.cv[0].cv_percent == 63.0
    st = S.strip_timings(back)
    assert st.rows[0].setup_time == 0.0 and st.rows[0].solve_time == 0.0 and st.rows[0].iterations == 70


def test_empty_report(tmp_path):
    base = str(tmp_path / "empty_test")
    S.emit_report(S.IterationReport(), "csv", base)
    txt = open(base + ".csv").read()
    assert txt.startswith("scenario,method,grid") and txt.count("\n") == 1
    assert S.parse_report_csv(base).rows == []


def test_text_table(tmp_path):
    rep = S.IterationReport()
    for pe in (100.0, 0.01):
        for grid in ("10x10", "20x20"):
            rep.rows.append(S.ReportRow("s", "ilu0", grid, pe, iterations=5, converged=True))
    base = str(tmp_path / "tt_test")
    S.emit_report(rep, "text-table", base)
    txt = open(base + ".txt").read()
    assert "10x10" in txt and "ilu0" in txt and txt.index("Pe = 100") < txt.index("Pe = 0.01")
    with pytest.raises(A.ConfigError):
        S.emit_report(rep, "yaml", base)


def test_malformed_csv(tmp_path):
    base = str(tmp_path / "bad")
    open(base + ".csv", "w").write("nope\n")
    with pytest.raises(A.IoError):
        S.parse_report_csv(base)
    with pytest.raises(A.IoError):
        S.parse_report_csv(str(tmp_path / "absent"))


@pytest.mark.gpu
def test_gpu_sweep_matches_oracle(gpu, orc):
    cfg = _pe_config()
    cfg.scenarios += [S.Scenario(name=f"amg@{pe}", nx=20, ny=20, n_c=3, pe=pe, method=m)
                      for m in ("cpr-amg", "cptr3-amg") for pe in (1e-2, 1.0, 1e2)]
    rg, ro = S.run_sweep(cfg, gpu), S.run_sweep(cfg, orc)
    _check_pe_report(S.IterationReport(rg.rows[:6], rg.cv[:2]))
    for a, b in zip(rg.rows, ro.rows):
        assert a.error == b.error == ""
        assert abs(a.iterations - b.iterations) <= 1, (a.scenario, a.iterations, b.iterations)
        assert a.converged == b.converged
    assert [(c.method, c.grid) for c in rg.cv] == [(c.method, c.grid) for c in ro.cv]
