"""Wire formats and run artifacts of the reference, byte-compatible (host-side, not timed).

* Binary wire (controls.cpp:20-45,229-288), little-endian:
    control : u32 channels, u64 steps, f64 t_start, f64 dt, then channel-major f64 samples
    matrix  : u64 rows, u64 cols, then column-major (re, im) f64 pairs
    vector  : u64 n, then (re, im) f64 pairs
  In the reference these are the in-process "messages" between subinterval tasks and the
  coordinator (ism.cpp:356-371,461-512).  On the device path nothing is serialised (the task
  results stay in HBM); these functions let a GPU run exchange controls and propagators with
  reference tooling.
* CSV controls (controls.cpp:183-227): header ``t,u_1,...``, one row per step at the step
  midpoint, ``%.17g``.
* Run artifacts of ``qoc run`` (tools/main.cpp:94-200): ``iterations.jsonl``,
  ``control.csv``, ``summary.json`` (format_version 1) and ``profiling.json``.
"""
from __future__ import annotations

import io
import json
import math
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .ism import ControlProblem, IsmRun, TimeGrid


def write_control_binary(u, grid: TimeGrid) -> bytes:
    """write_control_binary (controls.cpp:229-236); u is (C, K)."""
    u = np.asarray(u, dtype=np.float64)
    C, K = u.shape
    return struct.pack("<IQdd", C, K, grid.t_start, grid.dt) + u.astype("<f8").tobytes(order="C")


def read_control_binary(data: bytes):
    """read_control_binary (controls.cpp:238-246) -> (u (C, K), TimeGrid)."""
    if len(data) < 28:
        raise RuntimeError("unexpected end of binary stream")
    C, K, t0, dt = struct.unpack_from("<IQdd", data, 0)
    need = 28 + 8 * C * K
    if len(data) < need:
        raise RuntimeError("unexpected end of binary stream")
    u = np.frombuffer(data, dtype="<f8", count=C * K, offset=28).reshape(C, K).astype(np.float64)
    return u, TimeGrid(t0, dt, int(K))


def write_matrix_binary(m) -> bytes:
    """write_matrix_binary (controls.cpp:248-256): u64 rows, u64 cols, column-major (re, im)."""
    m = np.atleast_2d(np.asarray(m, dtype=np.complex128))
    rows, cols = m.shape
    body = np.ascontiguousarray(m.T).view(np.float64).astype("<f8").tobytes()
    return struct.pack("<QQ", rows, cols) + body


def read_matrix_binary(data: bytes) -> np.ndarray:
    if len(data) < 16:
        raise RuntimeError("unexpected end of binary stream")
    rows, cols = struct.unpack_from("<QQ", data, 0)
    if len(data) < 16 + 16 * rows * cols:
        raise RuntimeError("unexpected end of binary stream")
    v = np.frombuffer(data, dtype="<f8", count=2 * rows * cols, offset=16).astype(np.float64)
    return v.view(np.complex128).reshape(cols, rows).T.copy()


def write_vector_binary(v) -> bytes:
    """write_vector_binary (controls.cpp:271-277)."""
    v = np.asarray(v, dtype=np.complex128).reshape(-1)
    return struct.pack("<Q", v.size) + v.view(np.float64).astype("<f8").tobytes()


def read_vector_binary(data: bytes) -> np.ndarray:
    (n,) = struct.unpack_from("<Q", data, 0)
    if len(data) < 8 + 16 * n:
        raise RuntimeError("unexpected end of binary stream")
    return np.frombuffer(data, dtype="<f8", count=2 * n, offset=8).astype(np.float64).view(np.complex128).copy()


def _g17(x: float) -> str:
    """printf("%.17g") (controls.cpp:47-51)."""
    if math.isnan(x):
        return "nan"
    if math.isinf(x):
        return "inf" if x > 0 else "-inf"
    return "%.17g" % x


def write_control_csv(u, grid: TimeGrid) -> str:
    """write_control_csv (controls.cpp:183-192): rows at the step midpoints."""
    u = np.asarray(u, dtype=np.float64)
    C, K = u.shape
    out = io.StringIO()
    out.write("t" + "".join(f",u_{c}" for c in range(1, C + 1)) + "\n")
    for j in range(K):
        out.write(_g17(grid.node(j) + 0.5 * grid.dt))
        for c in range(C):
            out.write("," + _g17(float(u[c, j])))
        out.write("\n")
    return out.getvalue()


def read_control_csv(text: str, grid: TimeGrid) -> np.ndarray:
    """read_control_csv (controls.cpp:201-221)."""
    lines = text.splitlines()
    if not lines:
        raise RuntimeError("control CSV: missing header")
    if not lines[0].startswith("t,"):
        raise RuntimeError("control CSV: header must start with 't,'")
    C = lines[0].count(",")
    u = np.empty((C, grid.steps))
    for j in range(grid.steps):
        if j + 1 >= len(lines):
            raise RuntimeError(f"control CSV: expected {grid.steps} rows")
        cells = lines[j + 1].split(",")
        if len(cells) < C + 1:
            raise RuntimeError(f"control CSV: row {j} has too few columns")
        u[:, j] = [float(x) for x in cells[1:C + 1]]
    return u


def _num(x):
    return None if x is None or (isinstance(x, float) and math.isnan(x)) else x


def iteration_json(it) -> dict:
    """iteration_json (tools/main.cpp:100-116); per-task CPU timings are not measured on the
    device path (tasks = [], seconds from the CUDA-event device time)."""
    j = {"iteration": it.iteration, "objective": _num(it.objective)}
    if it.exact_objective is not None:
        j["exact_objective"] = it.exact_objective
    if it.error is not None:
        j["error"] = it.error
    j["task_values"] = [float(v) for v in it.task_values]
    j["tasks"] = [{"compute_seconds": t.compute_seconds, "serialize_seconds": t.serialize_seconds,
                   "bytes_sent": t.bytes_sent} for t in getattr(it, "tasks", [])]
    j["coordinator_seconds"] = 0.0
    j["critical_path_seconds"] = it.device_seconds
    j["instrumentation_seconds"] = 0.0
    j["wall_seconds"] = it.device_seconds
    j["events"] = list(getattr(it, "events", []))
    return j


def write_run_artifacts(directory, problem: ControlProblem, run: IsmRun, config: dict | None = None) -> None:
    """write_run_artifacts (tools/main.cpp:178-200) for a device run."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    rec = run.record
    if config is not None:
        (d / "config.json").write_text(json.dumps(config, indent=2) + "\n")
    (d / "iterations.jsonl").write_text("".join(json.dumps(iteration_json(it)) + "\n" for it in rec.iterations))
    (d / "control.csv").write_text(write_control_csv(run.control, problem.grid))
    g = problem.grid
    result = {"subintervals": rec.subintervals, "workers": rec.workers, "solver": rec.solver,
              "variant": rec.variant, "plan": rec.plan,
              "iterations": rec.iterations[-1].iteration if rec.iterations else 0,
              "aborted": rec.aborted, "abort_reason": rec.abort_reason,
              "total_wall_seconds": sum(it.device_seconds for it in rec.iterations),
              "total_critical_path_seconds": sum(it.device_seconds for it in rec.iterations)}
    if rec.iterations:
        last = rec.iterations[-1]
        result["final_objective"] = _num(last.objective)
        if last.exact_objective is not None:
            result["final_exact_objective"] = last.exact_objective
        if last.error is not None:
            result["final_error"] = last.error
    summary = {"format_version": 1, "config": config or {},
               "problem": {"state_dim": problem.model.state_dim(), "channels": problem.model.channels(),
                           "steps": g.steps, "t_start": g.t_start, "dt": g.dt, "duration": g.dt * g.steps},
               "result": result}
    (d / "summary.json").write_text(json.dumps(summary, indent=2) + "\n")
    secs = [it.device_seconds for it in rec.iterations]
    prof = {"entries": len(secs), "coordinator_seconds_total": 0.0,
            "critical_path_seconds_total": float(sum(secs)), "instrumentation_seconds_total": 0.0,
            "wall_seconds_total": float(sum(secs)), "max_task_seconds": 0.0, "bytes_sent_total": 0}
    if secs:
        prof["bootstrap_seconds"] = secs[0]
    (d / "profiling.json").write_text(json.dumps(prof, indent=2) + "\n")


# ---- speedup / efficiency reporting (runtime.cpp:117-174, tools/main.cpp:304-375) ------------
@dataclass
class EfficiencyRow:
    """runtime.hpp:83-89."""
    subintervals: int
    t_seconds: float = 0.0
    speedup: float = 0.0
    efficiency_percent: float = 0.0
    reached: bool = False


def _critical_path(it) -> float:
    v = getattr(it, "critical_path_seconds", None)
    return it.device_seconds if v is None else v


def time_to_target(record, limit_value: float, eps: float):
    """time_to_target (runtime.cpp:117-124): earliest cumulative critical-path time at which the
    recorded objective came within eps of limit_value; None if never."""
    cumulative = 0.0
    for it in record.iterations:
        cumulative += _critical_path(it)
        if limit_value - it.objective < eps:
            return cumulative
    return None


def efficiency_table(runs, limit_value: float, eps: float) -> list:
    """efficiency_table (runtime.cpp:126-153): runs = [(N, RunRecord)], speedups relative to
    the N = 1 entry, which must be present and reach the target."""
    base = None
    for n, rec in runs:
        if n == 1:
            base = time_to_target(rec, limit_value, eps)
            break
    if base is None:
        raise ValueError("efficiency table needs an N=1 run that reaches the target")
    rows = []
    for n, rec in runs:
        row = EfficiencyRow(subintervals=n)
        t = time_to_target(rec, limit_value, eps)
        row.reached = t is not None
        if t is not None:
            row.t_seconds = t
            row.speedup = base / t
            row.efficiency_percent = 100.0 * row.speedup / n
        rows.append(row)
    return rows


def format_percent(value: float) -> str:
    """format_percent (runtime.cpp:155-159): printf "%.1f%%"."""
    return "%.1f%%" % value


def efficiency_csv(rows) -> str:
    """efficiency_csv (runtime.cpp:161-174)."""
    out = "N,t_seconds,speedup,efficiency\n"
    for r in rows:
        if r.reached:
            out += "%d,%.6f,%.6f,%s\n" % (r.subintervals, r.t_seconds, r.speedup, format_percent(r.efficiency_percent))
        else:
            out += "%d,,,unreached\n" % r.subintervals
    return out


def bench_efficiency_csv(runs, eps_list) -> str:
    """The `qoc bench` efficiency.csv (tools/main.cpp:339-372): limit = best finite N = 1
    objective, one block of rows per eps ("eps,N,t_seconds,speedup,efficiency")."""
    limit = -math.inf
    for n, rec in runs:
        if n == 1:
            for it in rec.iterations:
                if math.isfinite(it.objective):
                    limit = max(limit, it.objective)
    if not math.isfinite(limit):
        raise ValueError("bench needs an N=1 run with a finite objective")
    csv = "eps,N,t_seconds,speedup,efficiency\n"
    for eps in eps_list:
        try:
            rows = efficiency_table(runs, limit, eps)
        except ValueError:
            continue
        for r in rows:
            if r.reached:
                csv += "%g,%d,%.6e,%.3f,%s\n" % (eps, r.subintervals, r.t_seconds, r.speedup,
                                                 format_percent(r.efficiency_percent))
            else:
                csv += "%g,%d,,,unreached\n" % (eps, r.subintervals)
    return csv
