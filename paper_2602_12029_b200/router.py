"""Model-aware prefill routing (drop-in for src/prefillsim/router.py) plus the
B200 placement map.

Semantics (bit-exact with the reference, checked against
tests/golden/router_traces.json):
  * baseline mode: model i's requests always go to prefill worker i and
    cache under that model's own namespace (router.py:53-56, :65-69);
  * prefillshare mode: every model shares one namespace; a session is routed
    once to the least-queued worker (ties -> lowest id) and stays pinned there
    for its whole life (router.py:58-77, RoutingTable :28-42);
  * decode worker of a model = n_models + its index (router.py:79-85);
  * unknown model ids raise ConfigurationError.

Placement (new, B200): the reference fleet has one logical prefill worker
and one decode worker per model. `Placement` maps those logical workers onto
GPUs (e.g. 2 prefill GPUs + 6 decode GPUs, or everything on one GPU) without
changing any routing decision.
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field

from .kvstore import SHARED_NS, model_ns


class ServingMode(enum.Enum):
    BASELINE = "baseline"
    PREFILLSHARE = "prefillshare"


class ConfigurationError(Exception):
    pass


@dataclass
class RoutingTable:
    """session id -> prefill worker; an entry is written once and never moves."""

    pins: dict[int, int] = field(default_factory=dict)

    def pin(self, session_id: int, worker_id: int) -> None:
        have = self.pins.get(session_id)
        if have is None:
            self.pins[session_id] = worker_id
        elif have != worker_id:
            raise RuntimeError(f"session {session_id} already pinned to worker {have}")

    def get(self, session_id: int) -> int | None:
        return self.pins.get(session_id)


class Router:
    def __init__(self, mode: ServingMode, model_ids: list[str]) -> None:
        self.mode = mode
        self.model_ids = list(model_ids)
        self.table = RoutingTable()
        self._index = {m: i for i, m in enumerate(self.model_ids)}

    def _model_index(self, model_id: str) -> int:
        try:
            return self._index[model_id]
        except KeyError:
            raise ConfigurationError(f"unknown model_id {model_id!r}") from None

    def prefill_namespace(self, model_id: str) -> str:
        return SHARED_NS if self.mode is ServingMode.PREFILLSHARE else model_ns(model_id)

    def route_prefill(self, request, queue_depths: list[int]) -> int:
        idx = self._model_index(request.model_id)
        if self.mode is ServingMode.BASELINE:
            return idx
        w = self.table.get(request.session_id)
        if w is None:
            # least queued, lowest id on ties
            w = min(range(len(queue_depths)), key=queue_depths.__getitem__)
            self.table.pin(request.session_id, w)
        return w

    def decode_worker(self, request) -> int:
        return len(self.model_ids) + self._model_index(request.model_id)


@dataclass(frozen=True)
class Placement:
    """Logical workers -> GPUs. prefill_gpus[i]: GPU of logical prefill worker
    i; decode_gpus[j]: GPU of model j's decode worker (its first replica).
    decode_replicas[j] (optional): every GPU holding a replica of model j's
    decode worker. The logical decode worker id stays n_models + j
    (router.py:79-85, bit-exact); which replica serves a request is a
    placement decision (the coordinator picks the one with the most free
    rows), so 2 prefill + 6 decode GPUs use all six decode GPUs for four
    models."""

    prefill_gpus: tuple[int, ...]
    decode_gpus: tuple[int, ...]
    decode_replicas: tuple[tuple[int, ...], ...] | None = None

    def replicas(self, model_index: int) -> tuple[int, ...]:
        if self.decode_replicas is None:
            return (self.decode_gpus[model_index],)
        return self.decode_replicas[model_index]

    def decode_models_on(self, gpu: int) -> list[int]:
        """Models with a decode replica on `gpu`."""
        return [m for m in range(len(self.decode_gpus)) if gpu in self.replicas(m)]

    @staticmethod
    def colocated(n_models: int, n_prefill: int | None = None, gpu: int = 0) -> "Placement":
        n_prefill = n_models if n_prefill is None else n_prefill
        return Placement((gpu,) * n_prefill, (gpu,) * n_models)

    @staticmethod
    def split(n_models: int, prefill_gpus: list[int], decode_gpus: list[int],
              n_prefill: int | None = None, replicate: bool = False) -> "Placement":
        """Round-robin logical workers over disjoint prefill / decode GPU sets
        (BASELINE.json config 3: 2 prefill GPUs + 6 decode GPUs). replicate:
        decode GPU k holds a replica of model k % n_models, so every decode
        GPU serves (with fewer decode GPUs than models, GPUs host several
        models as without replicas)."""
        n_prefill = n_models if n_prefill is None else n_prefill
        pre = tuple(prefill_gpus[i % len(prefill_gpus)] for i in range(n_prefill))
        first = tuple(decode_gpus[j % len(decode_gpus)] for j in range(n_models))
        if not replicate or len(decode_gpus) <= n_models:
            return Placement(pre, first)
        reps = tuple(tuple(g for k, g in enumerate(decode_gpus) if k % n_models == j) for j in range(n_models))
        return Placement(pre, first, reps)

    def handoff_is_local(self, prefill_worker: int, model_index: int) -> bool:
        return self.prefill_gpus[prefill_worker] == self.decode_gpus[model_index]
