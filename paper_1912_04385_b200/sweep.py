"""Sweep harness over the GPU solver (harness.{hpp,cpp}:13-400).

Same names, keys, formats and error behaviour as the reference's
`parse_config` / `run_sweep` / `compute_cv` / `emit_report` /
`parse_report_csv`; every solve goes through the C ABI (`mprec_gpu_*`).
Generated scenarios use this repository's seeded generator (`gen.py`, the
BASELINE recipe) in place of the reference's `build_problem`: grid, Peclet
(kappa = q_inj rho c_p / (Pe L), synth.cpp:35-38 with the ProblemSpec
defaults) and log-normal permeability sigma map onto it directly.
"""
from __future__ import annotations

import io
import math
import os
import time
from dataclasses import dataclass, field

from . import gen
from .api import ConfigError, IoError, MprecError, parse_method

# ProblemSpec defaults (synth.hpp:15-45) used by kappa_for_peclet
_Q_INJ, _RHO, _C_P, _LENGTH = 4.32, 3.1, 1.42, 0.35


def kappa_for_peclet(pe: float, q_inj=_Q_INJ, rho=_RHO, c_p=_C_P, length=_LENGTH) -> float:
    """synth.cpp:35-38."""
    if pe <= 0.0:
        raise ConfigError("target Peclet number must be positive")
    return q_inj * rho * c_p / (pe * length)


@dataclass
class Scenario:
    name: str = ""
    nx: int = 10
    ny: int = 10
    kappa: float = 50.0
    n_c: int = 12
    n_solid: int = 1
    time_fraction: float = 0.5
    pe: float = 0.0               # target Peclet; 0 keeps kappa
    perm_sigma: float = 0.0       # > 0 switches on a log-normal permeability field
    perm_span_decades: float = 0.0
    basename: str = ""            # non-empty: ingest <basename>.{mtx,layout,rhs}
    method: str = "ilu0"
    tol: float = 1e-8
    max_iter: int = 500


@dataclass
class ExperimentConfig:
    scenarios: list = field(default_factory=list)
    output_dir: str = "."
    seed: int = 1


@dataclass
class ReportRow:
    scenario: str = ""
    method: str = ""
    grid: str = ""
    pe: float = 0.0
    matrix_dim: int = 0
    nnz: int = 0
    iterations: int = 0
    converged: bool = False
    final_true_resid: float = 0.0
    setup_time: float = 0.0
    solve_time: float = 0.0
    error: str = ""


@dataclass
class CvRow:
    method: str
    grid: str
    cv_percent: float


@dataclass
class IterationReport:
    rows: list = field(default_factory=list)
    cv: list = field(default_factory=list)


def _to_double(v: str, key: str) -> float:
    try:
        return float(v)
    except ValueError:
        raise ConfigError(f"invalid number '{v}' for key {key}") from None


def _to_int(v: str, key: str) -> int:
    d = _to_double(v, key)
    if d != math.floor(d):
        raise ConfigError(f"key {key} needs an integer")
    return int(d)


_SCENARIO_KEYS = {"name": str, "nx": int, "ny": int, "pe": float, "kappa": float, "time_fraction": float,
                  "n_c": int, "n_solid": int, "perm_sigma": float, "perm_span_decades": float, "basename": str,
                  "method": str, "tol": float, "max_iter": int}


def parse_config_stream(text: str, origin: str) -> ExperimentConfig:
    """parse_config_stream (harness.cpp:47-122): `[sweep]` (seed, output) and
    one `[scenario]` section per entry; `;` / `#` comments."""
    cfg = ExperimentConfig()
    section = ""
    for lineno, line in enumerate(io.StringIO(text), start=1):
        for ch in ";#":
            p = line.find(ch)
            if p >= 0:
                line = line[:p]
        line = line.strip(" \t\r\n")
        if not line:
            continue
        where = f"{origin}:{lineno}"
        if line[0] == "[":
            if line[-1] != "]":
                raise ConfigError(f"unterminated section at {where}")
            section = line[1:-1].strip()
            if section == "scenario":
                cfg.scenarios.append(Scenario())
            elif section != "sweep":
                raise ConfigError(f"unknown section [{section}] at {where}")
            continue
        if "=" not in line:
            raise ConfigError(f"expected key = value at {where}")
        key, val = (s.strip(" \t") for s in line.split("=", 1))
        if section == "sweep":
            if key == "seed":
                cfg.seed = int(_to_double(val, key))
            elif key == "output":
                cfg.output_dir = val
            else:
                raise ConfigError(f"unknown sweep key '{key}' at {where}")
        elif section == "scenario":
            if key not in _SCENARIO_KEYS:
                raise ConfigError(f"unknown scenario key '{key}' at {where}")
            t = _SCENARIO_KEYS[key]
            setattr(cfg.scenarios[-1], key,
                    val if t is str else (_to_int(val, key) if t is int else _to_double(val, key)))
        else:
            raise ConfigError(f"key outside any section at {where}")
    if not cfg.scenarios:
        raise ConfigError(f"config {origin} defines no scenarios")
    for sc in cfg.scenarios:
        parse_method(sc.method)
        if not (0.0 < sc.tol < 1.0):
            raise ConfigError("scenario tol must lie in (0,1)")
        if sc.max_iter <= 0:
            raise ConfigError("scenario max_iter must be positive")
    return cfg


def parse_config(path: str) -> ExperimentConfig:
    """parse_config (harness.cpp:124-129)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError:
        raise ConfigError(f"cannot open config file {path}") from None
    return parse_config_stream(text, path)


def compute_cv(values) -> float:
    """Population standard deviation / mean, in percent (harness.cpp:131-140)."""
    values = list(values)
    if not values:
        raise ConfigError("CV of an empty list")
    mean = sum(values) / len(values)
    if mean == 0.0:
        raise ConfigError("CV undefined for zero mean")
    ss = sum((v - mean) * (v - mean) for v in values)
    return math.sqrt(ss / len(values)) / mean * 100.0


def compute_cv_sample(values) -> float:
    """Sample (n-1) variant (harness.cpp:142-151)."""
    values = list(values)
    if len(values) < 2:
        raise ConfigError("sample CV needs at least two values")
    mean = sum(values) / len(values)
    if mean == 0.0:
        raise ConfigError("CV undefined for zero mean")
    ss = sum((v - mean) * (v - mean) for v in values)
    return math.sqrt(ss / (len(values) - 1)) / mean * 100.0


def _system_for(api, sc: Scenario, seed: int):
    """The scenario's system: ingested, or generated on the BASELINE recipe."""
    if sc.basename:
        s = api.ingest(sc.basename + ".mtx", sc.basename + ".layout", sc.basename + ".rhs")
        return s, "file", sc.pe
    kappa = kappa_for_peclet(sc.pe) if sc.pe > 0.0 else sc.kappa
    nb = sc.n_c + sc.n_solid + 1  # (n_c + n_solid - 1) s-unknowns + P + T
    a, b, _ = gen.generate(gen.make_spec(sc.nx, sc.ny, nb, kappa, sc.perm_sigma, False, seed))
    s = api.system(a)
    s.b = b
    pe = sc.pe if sc.pe > 0.0 else kappa_for_peclet_inverse(kappa)
    return s, f"{sc.nx}x{sc.ny}", pe


def kappa_for_peclet_inverse(kappa: float) -> float:
    return _Q_INJ * _RHO * _C_P / (kappa * _LENGTH)


def run_sweep(config: ExperimentConfig, api) -> IterationReport:
    """run_sweep (harness.cpp:221-285) through `api` (the GPU library)."""
    report = IterationReport()
    for idx, sc in enumerate(config.scenarios):
        row = ReportRow(scenario=sc.name or f"scenario{idx}", method=sc.method)
        try:
            parse_method(sc.method)
            s, row.grid, row.pe = _system_for(api, sc, config.seed + idx)
            row.matrix_dim = s.a.dim
            row.nnz = s.a.nnzb * s.a.nb * s.a.nb  # to_scalar keeps every stored block entry
            t0 = time.perf_counter()
            s.setup(sc.method, s.b)
            t1 = time.perf_counter()
            r = s.solve(sc.tol, sc.max_iter)
            row.iterations, row.converged = r.iterations, bool(r.converged)
            row.final_true_resid = r.final_true_residual
            row.setup_time = r.setup_time_s if r.setup_time_s else t1 - t0
            row.solve_time = r.wall_time_s
            s.close()
        except MprecError as e:
            row.error = str(e)
        except Exception as e:  # noqa: BLE001 -- the reference records and continues
            row.error = f"unexpected: {e}"
        report.rows.append(row)
    groups = []
    for r in report.rows:
        if not r.error and (r.method, r.grid) not in groups:
            groups.append((r.method, r.grid))
    for (m, g) in groups:
        it = [float(r.iterations) for r in report.rows if not r.error and r.method == m and r.grid == g]
        if len(it) >= 2:
            report.cv.append(CvRow(m, g, compute_cv(it)))
    return report


ROW_HEADER = ("scenario,method,grid,pe,matrix_dim,nnz,iterations,converged,final_true_resid,"
              "setup_time,solve_time,error")


def _fmt(v: float) -> str:
    return "%.17g" % v


def emit_report(report: IterationReport, fmt: str, basename: str) -> None:
    """emit_report (harness.cpp:314-371): csv (+ _cv.csv) or text-table."""
    if fmt == "csv":
        try:
            with open(basename + ".csv", "w") as f:
                f.write(ROW_HEADER + "\n")
                for r in report.rows:
                    f.write(f"{r.scenario},{r.method},{r.grid},{_fmt(r.pe)},{r.matrix_dim},{r.nnz},{r.iterations},"
                            f"{1 if r.converged else 0},{_fmt(r.final_true_resid)},{_fmt(r.setup_time)},"
                            f"{_fmt(r.solve_time)},{r.error}\n")
            with open(basename + "_cv.csv", "w") as f:
                f.write("method,grid,cv_percent\n")
                for r in report.cv:
                    f.write(f"{r.method},{r.grid},{_fmt(r.cv_percent)}\n")
        except OSError:
            raise IoError(f"cannot write {basename}.csv") from None
        return
    if fmt != "text-table":
        raise ConfigError(f"unknown report format {fmt}")
    pes = sorted({r.pe for r in report.rows}, reverse=True)
    out = []
    for pe in pes:
        out.append("Pe = %g\n" % pe)
        out.append("  grid        method        dim      nnz    iters  conv  true_resid\n")
        for r in sorted((r for r in report.rows if r.pe == pe), key=lambda r: r.grid):
            if r.error:
                out.append("  %-10s  %-12s  failed: %s\n" % (r.grid, r.method, r.error))
            else:
                out.append("  %-10s  %-12s  %7d  %7d  %5d  %4s  %10.3e\n" % (
                    r.grid, r.method, r.matrix_dim, r.nnz, r.iterations, "yes" if r.converged else "no",
                    r.final_true_resid))
        out.append("\n")
    if report.cv:
        out.append("CV across Pe [%]\n")
        for r in report.cv:
            out.append("  %-12s  %-10s  %6.2f\n" % (r.method, r.grid, r.cv_percent))
    try:
        with open(basename + ".txt", "w") as f:
            f.write("".join(out))
    except OSError:
        raise IoError(f"cannot write {basename}.txt") from None


def parse_report_csv(basename: str) -> IterationReport:
    """parse_report_csv (harness.cpp:373-...): the inverse of emit_report(csv)."""
    report = IterationReport()
    if not os.path.exists(basename + ".csv"):
        raise IoError(f"cannot open {basename}.csv")
    with open(basename + ".csv") as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != ROW_HEADER:
        raise IoError(f"unexpected CSV header in {basename}.csv")
    for line in lines[1:]:
        if not line.strip():
            continue
        fl = line.split(",")
        if len(fl) != 12:
            raise IoError(f"malformed CSV row in {basename}.csv")
        report.rows.append(ReportRow(fl[0], fl[1], fl[2], _to_double(fl[3], "pe"), _to_int(fl[4], "matrix_dim"),
                                     _to_int(fl[5], "nnz"), _to_int(fl[6], "iterations"),
                                     _to_int(fl[7], "converged") != 0, _to_double(fl[8], "final_true_resid"),
                                     _to_double(fl[9], "setup_time"), _to_double(fl[10], "solve_time"), fl[11]))
    cvp = basename + "_cv.csv"
    if os.path.exists(cvp):
        with open(cvp) as f:
            cl = f.read().split("\n")
        if not cl or cl[0] != "method,grid,cv_percent":
            raise IoError(f"unexpected CV header in {cvp}")
        for line in cl[1:]:
            if line.strip():
                fl = line.split(",")
                if len(fl) != 3:
                    raise IoError(f"malformed CV row in {cvp}")
                report.cv.append(CvRow(fl[0], fl[1], _to_double(fl[2], "cv_percent")))
    return report


def strip_timings(report: IterationReport) -> IterationReport:
    """strip_timings (harness.cpp:415-421): zero only the timing columns."""
    rows = [ReportRow(**{**r.__dict__, "setup_time": 0.0, "solve_time": 0.0}) for r in report.rows]
    return IterationReport(rows, list(report.cv))
