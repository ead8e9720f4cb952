"""Sweep protocol of the reference (src/prefillsim/experiment.py:28, 86-173)
on the real engine: a (value x mode) grid over one axis, per-cell workload
seeds, auto-concurrency for arrival-rate sweeps, and the sweep table.

  * cell seed = mix_seed(run seed, axis index, the value's float64 bits)
    (experiment.py:86-104): both modes of a cell replay the same trace;
  * arrival_rate cells set the Poisson rate, max_concurrent_sessions cells
    set the admission cap;
  * auto-concurrency (arrival-rate sweeps only): the cell runs every cap of
    DEFAULT_CAP_GRID and keeps the report with the highest
    throughput_tok_per_s (first on ties), recording the chosen cap
    (experiment.py:107-131);
  * sweep_table: the reference's CSV, byte for byte (experiment.py:155-173).

The reference runs cells in a process pool over its virtual-time simulator;
here a cell is a real-time run on the GPU (cells run one after another).
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Callable

from . import workload as wl

SWEEP_AXES = ("arrival_rate", "max_concurrent_sessions")  # experiment.py:25
DEFAULT_CAP_GRID = (10, 20, 40, 80, 160)                  # experiment.py:28


@dataclass(frozen=True)
class SweepCell:
    axis: str
    value: float
    mode: str
    report: dict
    cap: int                       # the admission cap the report was run with (0 = unbounded)
    chosen_cap: int | None = None  # auto-concurrency choice


def cell_seed(run_seed: int, axis: str, value) -> int:
    """experiment.py:89-90: float bit pattern, not hash() (process-randomized)."""
    bits = int.from_bytes(struct.pack(">d", float(value)), "big")
    return wl.mix_seed(run_seed, SWEEP_AXES.index(axis), bits)


def cell_workload(base: wl.WorkloadConfig, run_seed: int, axis: str, value) -> tuple[wl.WorkloadConfig, int]:
    """(workload config, admission cap) of one cell (experiment.py:86-104)."""
    if axis not in SWEEP_AXES:
        raise ValueError(f"unknown sweep axis {axis!r} (expected one of {SWEEP_AXES})")
    seed = cell_seed(run_seed, axis, value)
    if axis == "arrival_rate":
        return wl.WorkloadConfig(**{**base.__dict__, "arrival_rate_per_s": float(value), "seed": seed}), 0
    return wl.WorkloadConfig(**{**base.__dict__, "seed": seed}), int(value)


def run_cell(run: Callable[[list, str, int], dict], base: wl.WorkloadConfig, run_seed: int, axis: str, value,
             mode: str, cap_grid: tuple[int, ...] | None = None, default_cap: int = 0) -> SweepCell:
    """One cell. run(sessions, mode, cap) serves the sessions on the engine
    and returns a report.json dict (serve.build_report)."""
    wcfg, cap = cell_workload(base, run_seed, axis, value)
    if axis == "arrival_rate":
        cap = default_cap
    sessions = wl.generate(wcfg)
    if cap_grid is None:
        return SweepCell(axis, float(value), mode, run(sessions, mode, cap), cap)
    if axis != "arrival_rate":
        raise ValueError("auto-concurrency applies to arrival_rate sweeps only")
    best, best_cap = None, None
    for c in cap_grid:
        rep = run(sessions, mode, c)
        if best is None or rep["throughput_tok_per_s"] > best["throughput_tok_per_s"]:
            best, best_cap = rep, c
    best = dict(best, auto_concurrency_cap=best_cap)
    return SweepCell(axis, float(value), mode, best, best_cap, best_cap)


def run_sweep(run, base: wl.WorkloadConfig, run_seed: int, axis: str, values, modes,
              auto_concurrency: bool = False, cap_grid: tuple[int, ...] = DEFAULT_CAP_GRID,
              default_cap: int = 0) -> list[SweepCell]:
    """The (value x mode) grid in the reference's canonical order."""
    if not values:
        raise ValueError("sweep values must be non-empty")
    if auto_concurrency and axis != "arrival_rate":
        raise ValueError("--auto-concurrency applies to arrival_rate sweeps only")
    return [run_cell(run, base, run_seed, axis, v, m, cap_grid if auto_concurrency else None, default_cap)
            for v in values for m in modes]


def sweep_table(cells: list[SweepCell]) -> str:
    """experiment.py:155-173."""
    lines = ["axis,value,mode,cap,throughput_tok_per_s,p95_e2e_us,mean_ttft_us,prefix_hit_ratio,failures"]
    for cell in cells:
        r = cell.report
        cap = cell.chosen_cap if cell.chosen_cap is not None else cell.cap
        p95 = r["p95_e2e_us"] if r["p95_e2e_us"] is not None else ""
        ttft = r["mean_ttft_us"] if r["mean_ttft_us"] is not None else ""
        lines.append(f"{cell.axis},{cell.value:g},{cell.mode},{cap},{r['throughput_tok_per_s']:.3f},{p95},{ttft},"
                     f"{r['prefix_hit_ratio']:.6f},{r['failure_count']}")
    return "\n".join(lines) + "\n"
