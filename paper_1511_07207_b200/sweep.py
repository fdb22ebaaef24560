"""Benchmark sweeps and reports for the B200 path.

Keeps the reference's sweep API (harness.py:58-68 ``BenchRecord``, :261-305
``run_benchmark``, :312-372 ``emit_report`` / ``parse_report_csv``, the CSV column
contract) but measures the way a device backend should be measured:

* each (method, n, precision) point is generated once (the reference's seeded
  generators) and, for ``"b200"``, staged to the device ONCE: the timed solves read
  device-resident operands, so the record is solver time, not PCIe time.  The staging
  time is kept separately (``SweepPoint.stage_s``);
* every backend gets one untimed warm-up solve, then ``repeats`` synchronised solves;
  the record keeps the best (the reference's best-of protocol) and the median is kept
  beside it;
* the backend list may name the reference's own CPU backends (``"reference"``,
  ``"blocked"``) when the unmodified reference package is importable: those points run
  through the reference's ``solve_system``, so a b200-vs-reference speedup table comes
  out of one call;
* a solve that raises a ``LinAlgError`` is recorded as a NaN row and the sweep goes on.
"""

from __future__ import annotations

import dataclasses
import io
import math
import statistics
import time
from dataclasses import dataclass

import numpy as np

from .core import LinAlgError, SolverConfig

CSV_COLUMNS = ("method", "n", "precision", "backend", "wall_time_s", "iterations", "converged",
               "relative_residual", "speedup")


@dataclass
class BenchRecord:
    """One (method, n, precision, backend) measurement (harness.py:58-68)."""
    method: str
    n: int
    precision: str
    backend: str
    wall_time: float
    iterations: int
    converged: bool
    relative_residual: float
    speedup_vs_reference: float


@dataclass
class SweepPoint:
    """Device-side detail of a b200 record (not part of the CSV contract)."""
    record: BenchRecord
    median_s: float
    stage_s: float


class _B200Runner:
    name = "b200"

    def __init__(self, backend):
        self.be = backend
        self.points: list[SweepPoint] = []

    def run(self, method, A, b, cfg, repeats):
        from .harness import solve_system
        t0 = time.perf_counter()
        dA, db = self.be.stage_in(A, b)
        self.be.ctx.synchronize()
        stage = time.perf_counter() - t0

        def once():
            return solve_system(method, dA, db, None, cfg, self.be)

        x, rep = once()  # warm-up; its report is the record's
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            once()  # returns after the device finished (the report is host data)
            times.append(time.perf_counter() - t0)
        return rep, times, stage


class _ReferenceRunner:
    """A CPU backend of the unmodified reference (baseline/_ref or an installed densolve)."""

    def __init__(self, name):
        import densolve  # noqa: PLC0415 - optional, only when the caller names a reference backend
        self.ds = densolve
        self.name = name
        self.be = densolve.get_backend(name)

    def run(self, method, A, b, cfg, repeats):
        ref_cfg = self.ds.SolverConfig(**{f.name: getattr(cfg, f.name) for f in dataclasses.fields(cfg)})

        def once():
            return self.ds.harness.solve_system(method, A, b, None, ref_cfg, self.be)

        try:
            x, rep = once()
        except self.ds.LinAlgError as e:
            raise LinAlgError(str(e)) from e
        times = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            once()
            times.append(time.perf_counter() - t0)
        return rep, times, 0.0


def _runner(name, cache):
    if name not in cache:
        if name == "b200":
            from .backends import get_backend
            cache[name] = _B200Runner(get_backend("b200"))
        else:
            try:
                cache[name] = _ReferenceRunner(name)
            except (ImportError, ValueError) as e:
                raise ValueError(f"unknown backend {name!r}: only 'b200', or a reference CPU backend when "
                                 f"the reference package is importable ({e})") from e
    return cache[name]


def _nan_record(method, n, precision, backend):
    return BenchRecord(method=method, n=n, precision=precision, backend=backend, wall_time=math.nan,
                       iterations=0, converged=False, relative_residual=math.nan,
                       speedup_vs_reference=math.nan)


def run_benchmark(methods, sizes, precisions, backends, cfg: SolverConfig, seed: int = 0,
                  repeats: int = 3) -> list[BenchRecord]:
    """Sweep methods x sizes x precisions over the named backends; speedups are relative to
    the first backend that solved the point.  ``points`` of the b200 runner keep the
    median and staging times (``run_benchmark.last_points``)."""
    from .harness import ALL_METHODS, METHOD_FAMILY, OUT_OF_SCOPE_METHODS, ProblemSpec, generate_problem

    if not (methods and sizes and precisions and backends):
        raise ValueError("methods, sizes, precisions and backends must be non-empty")
    for m in methods:
        if m in OUT_OF_SCOPE_METHODS:
            raise NotImplementedError(f"method {m!r} is not on the B200 hot path (SURVEY.md §8)")
        if m not in ALL_METHODS:
            raise ValueError(f"unknown method {m!r}")
    runners: dict = {}
    out: list[BenchRecord] = []
    points: list[SweepPoint] = []
    for method in methods:
        for n in sizes:
            for precision in precisions:
                A, b, _ = generate_problem(ProblemSpec(kind=METHOD_FAMILY[method], n=n, seed=seed,
                                                       precision=precision))
                base = None
                for name in backends:
                    r = _runner(name, runners)
                    try:
                        rep, times, stage = r.run(method, A, b, cfg, max(1, repeats))
                    except LinAlgError:
                        out.append(_nan_record(method, n, precision, name))
                        continue
                    best = min(times)
                    base = best if base is None else base
                    rec = BenchRecord(method=method, n=n, precision=precision, backend=name, wall_time=best,
                                      iterations=rep.iterations, converged=bool(rep.converged),
                                      relative_residual=float(rep.final_relative_residual),
                                      speedup_vs_reference=base / best)
                    out.append(rec)
                    if name == "b200":
                        points.append(SweepPoint(rec, statistics.median(times), stage))
    run_benchmark.last_points = points
    return out


run_benchmark.last_points = []


# ---- reports ------------------------------------------------------------------------------
def _csv_cell(v) -> str:
    if isinstance(v, bool):
        return "True" if v else "False"
    if isinstance(v, (float, np.floating)):
        return repr(float(v))
    return str(v)


def emit_report(records, format: str = "csv") -> str:
    """CSV (the reference's columns, round-trips through ``parse_report_csv``) or a
    markdown speedup grid per precision (sizes down, methods across; each cell
    "speedup x (best wall ms)" of the last backend measured at that point)."""
    if not records:
        raise ValueError("empty record list: nothing to report")
    if format == "csv":
        lines = [",".join(CSV_COLUMNS)]
        for r in records:
            row = (r.method, r.n, r.precision, r.backend, r.wall_time, r.iterations, r.converged,
                   r.relative_residual, r.speedup_vs_reference)
            lines.append(",".join(_csv_cell(v) for v in row))
        return "\n".join(lines) + "\n"
    if format == "markdown":
        return _markdown(records)
    raise ValueError(f"unknown report format {format!r}")


def _markdown(records) -> str:
    from .harness import ALL_METHODS

    buf = io.StringIO()
    for prec in sorted({r.precision for r in records}):
        recs = [r for r in records if r.precision == prec]
        first = recs[0].backend
        methods = sorted({r.method for r in recs}, key=ALL_METHODS.index)
        cell = {}
        for r in recs:  # the last backend listed wins the cell (the measured one vs the baseline)
            cell[(r.n, r.method)] = r
        buf.write(f"### {prec}: speedup vs {first} (best wall time)\n\n")
        buf.write("| Matrix dimension | " + " | ".join(methods) + " |\n")
        buf.write("|" + "---|" * (len(methods) + 1) + "\n")
        for n in sorted({r.n for r in recs}):
            row = []
            for m in methods:
                r = cell.get((n, m))
                row.append("-" if r is None or not r.wall_time == r.wall_time
                           else f"{r.speedup_vs_reference:.2f}x ({1e3 * r.wall_time:.3g} ms)")
            buf.write(f"| {n} | " + " | ".join(row) + " |\n")
        buf.write("\n")
    return buf.getvalue()


def parse_report_csv(text: str) -> list[BenchRecord]:
    lines = [ln for ln in text.splitlines() if ln.strip()]
    if not lines or tuple(lines[0].split(",")) != CSV_COLUMNS:
        raise ValueError("bad csv report header")
    out = []
    for ln in lines[1:]:
        f = ln.split(",")
        if len(f) != len(CSV_COLUMNS):
            raise ValueError(f"bad csv report row: {ln!r}")
        out.append(BenchRecord(method=f[0], n=int(f[1]), precision=f[2], backend=f[3], wall_time=float(f[4]),
                               iterations=int(f[5]), converged=f[6] == "True", relative_residual=float(f[7]),
                               speedup_vs_reference=float(f[8])))
    return out

