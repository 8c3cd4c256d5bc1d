"""The bench reporting format: the reference's
ResultRow schema and its CSV / JSON writers (include/phiact/bench.hpp:32-58,
proj/src/bench.cpp:37-57, 222-265), plus the one reference experiment on
this path, the ADR integrator order study (bench.cpp:131-179), run through
the device integrator (phx_integrate).

Formats, byte for byte like the reference's:
  * CSV: header "experiment,label,t,error,order,seconds,s_eff,series_len_S,
    sweeps,matvecs,bound,ok"; doubles as an ostream with precision(17)
    prints them (%.17g: "nan", "inf"); ok as 1/0;
  * JSON: nlohmann::json dump(2) of an array of objects -- keys in
    std::map (sorted) order, "order" / "bound" present only when finite,
    shortest round-trip doubles, two-space indent, trailing newline.
"""
from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import (ADRProblem, RunRecord, adr_build, default_tolerance, integrate,
               select_parameters)

__all__ = ["BenchConfig", "ResultRow", "make_row", "rows_to_csv", "rows_to_json", "write_rows",
           "all_within_bounds", "run_adr"]


@dataclass
class BenchConfig:  # bench.hpp:15-29 (the fields the ADR study reads)
    experiment: str = "adr"
    adr_nx: int = 50
    adr_ny: int = 50
    tol: float = -1.0  # <= 0: per-experiment default
    m: int = 61
    delta: float = 0.8
    out_path: str = ""
    format: str = "csv"


@dataclass
class ResultRow:  # bench.hpp:32-47
    experiment: str = ""
    label: str = ""
    t: float = 0.0
    error: float = 0.0
    order: float = math.nan
    seconds: float = 0.0
    s_effective: int = 0
    series_len_S: int = 0
    sweeps: int = 0
    matvecs: int = 0
    bound: float = math.nan
    ok: bool = True


def make_row(experiment, label, t, error, seconds, rec: RunRecord, bound) -> ResultRow:
    """bench.cpp:39-57; ok = !(error > bound), so a NaN bound never fails."""
    return ResultRow(experiment, label, float(t), float(error), math.nan, float(seconds),
                     int(rec.s_effective), int(rec.series_len_S), len(rec.series_lens_F),
                     int(rec.matvecs), float(bound), not (error > bound))


def _g17(x: float) -> str:
    return format(float(x), ".17g")


def rows_to_csv(rows) -> str:  # bench.cpp:222-234
    out = ["experiment,label,t,error,order,seconds,s_eff,series_len_S,sweeps,matvecs,bound,ok\n"]
    for r in rows:
        out.append(",".join([r.experiment, r.label, _g17(r.t), _g17(r.error), _g17(r.order),
                             _g17(r.seconds), str(int(r.s_effective)), str(int(r.series_len_S)),
                             str(int(r.sweeps)), str(int(r.matvecs)), _g17(r.bound),
                             "1" if r.ok else "0"]) + "\n")
    return "".join(out)


def rows_to_json(rows) -> str:  # bench.cpp:236-255
    arr = []
    for r in rows:
        obj = {"experiment": r.experiment, "label": r.label, "t": float(r.t),
               "error": float(r.error), "seconds": float(r.seconds),
               "s_eff": int(r.s_effective), "series_len_S": int(r.series_len_S),
               "sweeps": int(r.sweeps), "matvecs": int(r.matvecs), "ok": bool(r.ok)}
        if math.isfinite(r.order):
            obj["order"] = float(r.order)
        if math.isfinite(r.bound):
            obj["bound"] = float(r.bound)
        arr.append(obj)
    return json.dumps(arr, indent=2, sort_keys=True) + "\n"


def write_rows(rows, cfg: BenchConfig) -> None:  # bench.cpp:257-263
    if not cfg.out_path:
        return
    try:
        with open(cfg.out_path, "w") as f:
            f.write(rows_to_json(rows) if cfg.format == "json" else rows_to_csv(rows))
    except OSError as e:
        raise RuntimeError("cannot open output file " + cfg.out_path) from e


def all_within_bounds(rows) -> bool:  # bench.cpp:265-269
    return all(r.ok for r in rows)


def _rel_err_inf(got, want) -> float:
    d = float(np.abs(want).max()) if np.size(want) else 0.0
    e = float(np.abs(np.asarray(got) - np.asarray(want)).max()) if np.size(want) else 0.0
    return e / d if d > 0.0 else e


def run_adr(cfg: BenchConfig, device: int = -1) -> list:
    """The ADR convergence study (bench.cpp:131-179) on the device integrator:
    T = t_end/16, h0 = T/128, h in {h0, h0/2, h0/4, h0/8} against a reference
    run at h0/128 with the default tolerance; observed order on each row after
    the first, ok = order >= 3.5."""
    tol = cfg.tol if cfg.tol > 0.0 else 1e-7
    problem: ADRProblem = adr_build(cfg.adr_nx, cfg.adr_ny, device=device)
    params = select_parameters(problem.op, cfg.m, tol, cfg.delta)
    t_end = problem.t_end / 16.0
    h0 = t_end / 128.0
    hs = [h0, h0 / 2.0, h0 / 4.0, h0 / 8.0]
    ref_params = select_parameters(problem.op, cfg.m, default_tolerance(), cfg.delta)
    ref = integrate(problem, hs[-1] / 16.0, t_end, default_tolerance(), ref_params,
                    keep_records=False)
    rows = []
    prev_err = 0.0
    for i, h in enumerate(hs):
        start = time.perf_counter()
        res = integrate(problem, h, t_end, tol, params)
        elapsed = time.perf_counter() - start
        err = _rel_err_inf(res.u, ref.u)
        agg = RunRecord()
        for step in res.steps:
            for call in step.calls:
                agg.s_effective = max(agg.s_effective, call.s_effective)
                agg.series_len_S = max(agg.series_len_S, call.series_len_S)
                agg.matvecs += call.matvecs
        row = make_row("adr", f"grid={cfg.adr_nx}", h, err, elapsed, agg, math.nan)
        if i > 0:
            row.order = math.log2(prev_err / err)
            row.ok = row.order >= 3.5
        prev_err = err
        rows.append(row)
    return rows
