"""Seeded multi-model agent workloads (restates src/prefillsim/workload.py;
checked against tests/golden/workload.json produced by the reference).

Poisson session arrivals from a splitmix64 stream by inverse CDF, agent
chains rotated round-robin per session, and synthetic 64-bit token ids
packed as (session+1, purpose, index) so sessions never share prefixes
(workload.py:6-8, :142-154). Kept in Python on purpose: arrival times use
float64 log and Python's round-half-even exactly like the reference
(workload.py:99, :109).
"""

from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Iterator

M64 = 0xFFFFFFFFFFFFFFFF
GOLDEN = 0x9E3779B97F4A7C15

PATTERN_PRESETS = {  # (prompt, extension, output, turns) per workload.py:24-27
    "react": {"initial_prompt_len": 512, "input_extension_len": 64, "output_len": 128, "turns": 3},
    "reflexion": {"initial_prompt_len": 512, "input_extension_len": 96, "output_len": 256, "turns": 3},
}
DEFAULT_MODELS = ("model_a", "model_b", "model_c", "model_d")


def _finalize(z: int) -> int:
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return z ^ (z >> 31)


def splitmix64(state: int) -> Iterator[int]:
    s = state & M64
    while True:
        s = (s + GOLDEN) & M64
        yield _finalize(s)


def mix_seed(*parts: int) -> int:
    acc = 0x243F6A8885A308D3
    for p in parts:
        acc = _finalize(((acc ^ (p & M64)) + GOLDEN) & M64)
    return acc


@dataclass(frozen=True)
class AgentProfile:
    model_id: str
    input_extension_len: int
    output_len: int

    def __post_init__(self):
        if self.output_len < 1:
            raise ValueError("output_len must be >= 1")
        if self.input_extension_len < 0:
            raise ValueError("input_extension_len must be >= 0")


@dataclass(frozen=True)
class SessionSpec:
    session_id: int
    arrival_time: int       # microseconds
    initial_prompt_len: int
    turns: int
    agent_chain: tuple

    @property
    def total_requests(self) -> int:
        return self.turns * len(self.agent_chain)


@dataclass(frozen=True)
class WorkloadConfig:
    pattern: str = "react"
    arrival_rate_per_s: float = 4.0
    duration_s: float = 60.0
    seed: int = 0
    initial_prompt_len: int | None = None
    turns: int | None = None
    agents: tuple | None = None

    def __post_init__(self):
        if self.pattern not in PATTERN_PRESETS:
            raise ValueError(f"unknown pattern {self.pattern!r}")
        if not self.arrival_rate_per_s > 0 or not self.duration_s > 0:
            raise ValueError("arrival_rate_per_s and duration_s must be > 0")

    def chain(self) -> tuple:
        p = PATTERN_PRESETS[self.pattern]
        if self.agents is not None:
            return tuple(AgentProfile(m, e, o) for m, e, o in self.agents)
        return tuple(AgentProfile(m, p["input_extension_len"], p["output_len"]) for m in DEFAULT_MODELS)


def generate(cfg: WorkloadConfig) -> list[SessionSpec]:
    """workload.py:96-125."""
    p = PATTERN_PRESETS[cfg.pattern]
    chain = cfg.chain()
    turns = p["turns"] if cfg.turns is None else cfg.turns
    prompt = p["initial_prompt_len"] if cfg.initial_prompt_len is None else cfg.initial_prompt_len
    horizon = int(round(cfg.duration_s * 1_000_000))
    rng = splitmix64(cfg.seed)
    out: list[SessionSpec] = []
    t = 0
    while True:
        u = (next(rng) + 1) / 2.0 ** 64  # (0, 1]
        t += int(round(-math.log(u) / cfg.arrival_rate_per_s * 1_000_000))
        if t > horizon:
            return out
        k = len(out) % len(chain)
        out.append(SessionSpec(len(out), t, prompt, turns, chain[k:] + chain[:k]))


def prompt_slot() -> int:
    return 0


def extension_slot(i: int) -> int:
    return 2 * i + 1


def output_slot(i: int) -> int:
    return 2 * i + 2


def synth_base(session_id: int, purpose: int) -> int:
    return ((session_id + 1) << 32) | (purpose << 16)


def synth_tokens(session_id: int, purpose: int, length: int) -> tuple:
    if length < 0:
        raise ValueError("length must be >= 0")
    if length > 1 << 16 or purpose >= 1 << 16:
        raise ValueError("length/purpose exceed the packing limits")
    b = synth_base(session_id, purpose)
    return tuple(range(b, b + length))


def export_sessions(sessions: list[SessionSpec]) -> str:
    return json.dumps({"schema_version": 1, "sessions": [
        {"session_id": s.session_id, "arrival_time_us": s.arrival_time,
         "initial_prompt_len": s.initial_prompt_len, "turns": s.turns,
         "agents": [[a.model_id, a.input_extension_len, a.output_len] for a in s.agent_chain]}
        for s in sessions]}, sort_keys=True, indent=1)


def import_sessions(text: str) -> list[SessionSpec]:
    return [SessionSpec(d["session_id"], d["arrival_time_us"], d["initial_prompt_len"], d["turns"],
                        tuple(AgentProfile(*a) for a in d["agents"]))
            for d in json.loads(text)["sessions"]]
