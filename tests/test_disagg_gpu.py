"""Disaggregated serving on one B200 (roles co-located, world_size 1): the
real backends (GPU BlockPool, batched prefill K1-K3, K8 page-copy handoff,
CUDA-graph decode steps with K5/K6) through the disagg.py round protocol."""

import os
import socket

import pytest
import torch
import torch.distributed as dist

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode_name", ["prefillshare", "baseline"])
def test_disagg_colocated_tiny(mode_name):
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.disagg import (Coordinator, DisaggServer, GpuDecodeBackend, GpuPrefillBackend,
                                              summarize)
    from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights
    from paper_2602_12029_b200.router import Placement, Router, ServingMode
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        mode = ServingMode(mode_name)
        models = list(wl.DEFAULT_MODELS)
        cfg = LlamaConfig.tiny(max_pos=4096)
        n_prefill = 4 if mode is ServingMode.BASELINE else 1
        place = Placement.colocated(4, n_prefill)
        mods = {m: ModuleWeights(cfg, 10 + m) for m in range(4)}
        base = ModuleWeights(cfg, 9, with_head=False)
        prefill = {w: GpuPrefillBackend(cfg, base if mode is ServingMode.PREFILLSHARE else mods[w], 1024, 4096, 64)
                   for w in range(n_prefill)}
        decode = GpuDecodeBackend(cfg, mods, rows_per_model=3, ctx_pages=3 * 4 * 200, max_context=4096,
                                  max_output=128)
        srv = DisaggServer(place, models, mode, prefill, decode, rows_per_model=3)
        sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=4.0, duration_s=1.0, seed=1,
                                                 turns=2))
        coord = Coordinator(sessions, models, Router(mode, models), place, time_scale=0.1, steps_per_round=16)
        recs = srv.run(coord)
        torch.cuda.synchronize()
        n_req = sum(s.total_requests for s in sessions)
        assert len(recs) == n_req
        assert all(r.done_us is not None and not r.failed and r.out_tokens == 128 for r in recs.values())
        s = summarize(recs)
        assert s["completed"] == n_req
        if mode is ServingMode.PREFILLSHARE:
            assert s["prefix_hit_ratio"] > 0.3
    finally:
        dist.destroy_process_group()


def test_bench_pd_split_point_colocated_tiny():
    """bench.pd_split_point end to end on one GPU (tiny shape, every role
    co-located, world 1): both modes served, stats gathered, memory freed.
    The N-GPU NCCL path differs only in the handoff transport (gloo-tested
    at world 3/4 in test_disagg.py)."""
    import bench
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.model import LlamaConfig
    from paper_2602_12029_b200.router import Placement
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        cfg = LlamaConfig.tiny(max_pos=4096 + 512)
        out = bench.pd_split_point(1, 0, 0, None, duration=1.0, rows=4, pool_pages=1024, cfg=cfg,
                                   place=Placement.colocated(len(wl.DEFAULT_MODELS)), max_context=4096,
                                   max_output=256)
        for mode in ("baseline", "prefillshare"):
            assert out[mode]["completed"] > 0 and out[mode]["failed"] == 0
            assert out[mode]["handoff"]["bytes"] == 0  # co-located: page copies, no P2P
        assert out["prefillshare"]["prefix_hit_ratio"] > out["baseline"]["prefix_hit_ratio"]
        assert "req_per_s_ratio" in out
    finally:
        dist.destroy_process_group()
