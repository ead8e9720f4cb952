"""Disaggregated serving (disagg.py) of the agent workload on N GPUs, one
process per GPU (BASELINE config 3: P prefill GPUs + N-P decode GPUs; on one
GPU the roles are co-located and the handoff is a K8 page copy).

    torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/run_disagg.py \
        [--prefill-gpus P] [--mode prefillshare|baseline] [--rate 8] [--duration 20]
    python tools/run_disagg.py ...            # 1 GPU
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_12029_b200 import workload as wl  # noqa: E402
from paper_2602_12029_b200.disagg import (Coordinator, DisaggServer, GpuDecodeBackend,  # noqa: E402
                                          GpuPrefillBackend, summarize)
from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights  # noqa: E402
from paper_2602_12029_b200.router import Placement, Router, ServingMode  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="8b")
    ap.add_argument("--mode", default="prefillshare")
    ap.add_argument("--rate", type=float, default=8.0)
    ap.add_argument("--duration", type=float, default=20.0)
    ap.add_argument("--pattern", default="react")
    ap.add_argument("--prefill-gpus", type=int, default=None)
    ap.add_argument("--rows", type=int, default=64, help="decode rows per model")
    ap.add_argument("--pool-pages", type=int, default=7500, help="per prefill worker")
    ap.add_argument("--steps-per-round", type=int, default=8)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-context", type=int, default=None)
    a = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29611")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", local))
        data = None
    else:
        dist.init_process_group("gloo", rank=0, world_size=1)
        data = None
    ctrl = dist.new_group(backend="gloo")
    mode = ServingMode(a.mode)
    models = list(wl.DEFAULT_MODELS)
    M = len(models)
    # longest context: react 4096, reflexion 512 + 12 x (96 + 256) = 4736 (as run_agents.py)
    max_ctx = a.max_context or (5120 if a.pattern == "reflexion" else 4096)
    cfg = (LlamaConfig.llama8b(max_pos=max_ctx + 512) if a.shape == "8b"
           else LlamaConfig.tiny(max_pos=max_ctx + 512))
    # the reference fleet: one logical prefill worker (own pool) per model in
    # both modes (cluster.py:156-160), placed round-robin on the prefill GPUs
    n_prefill = M
    if world == 1:
        place = Placement.colocated(M, n_prefill)
    else:
        P = a.prefill_gpus or max(1, world // 4)
        place = Placement.split(M, list(range(P)), list(range(P, world)), n_prefill, replicate=True)
    mine_p = [w for w, r in enumerate(place.prefill_gpus) if r == rank]
    mine_d = place.decode_models_on(rank)
    base = ModuleWeights(cfg, 99, with_head=False, device=local) if (mine_p and mode is ServingMode.PREFILLSHARE) else None
    mods = {m: ModuleWeights(cfg, 100 + m, device=local) for m in set(mine_d) | (set(mine_p) if mode is ServingMode.BASELINE else set())}
    prefill = {w: GpuPrefillBackend(cfg, base if base is not None else mods[w], a.pool_pages, max_ctx, 256, local)
               for w in mine_p}
    decode = (GpuDecodeBackend(cfg, {m: mods[m] for m in mine_d}, a.rows, ctx_pages=len(mine_d) * a.rows * (max_ctx // 16 + 4),
                               max_context=max_ctx, max_output=256, device=local) if mine_d else None)
    srv = DisaggServer(place, models, mode, prefill, decode, a.rows, ctrl_group=ctrl, data_group=data)
    coord = None
    if rank == 0:
        sessions = wl.generate(wl.WorkloadConfig(pattern=a.pattern, arrival_rate_per_s=a.rate,
                                                 duration_s=a.duration, seed=a.seed))
        coord = Coordinator(sessions, models, Router(mode, models), place, steps_per_round=a.steps_per_round)
    recs = srv.run(coord)
    if rank == 0:
        out = {"mode": a.mode, "gpus": world, "placement": {"prefill": list(place.prefill_gpus),
                                                           "decode": [list(place.replicas(m)) for m in range(M)]},
               "workload": {"pattern": a.pattern, "rate": a.rate, "duration_s": a.duration,
                            "sessions": len(sessions), "requests": sum(s.total_requests for s in sessions)},
               "summary": summarize(recs)}
        print(json.dumps(out))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
