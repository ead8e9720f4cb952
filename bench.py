"""PrefillShare hot-path benchmark (BASELINE.json configs[1]).

Workload (N=1): Llama-3.1-8B-shape frozen prefill module + 4 decode modules
(random init, bf16) on one B200. One step = one serve() of a batch of
--sessions concurrent agent sessions (default 32), each a fresh synthetic
4096-token prompt: GPU block-pool lookup/insert (K7), shared prefill of each
prompt (K1-K3), then every decode module generates 256 tokens greedily from
the shared KV (K5/K5-TC GEMV, K6 attention), all sessions x modules
co-batched in one decode step.
A request = one decode module's 256-token generation on one session; its
latency is the serve() duration. Other batch sizes (S = 1, the latency-optimal
point, 8 and 64) are reported under "sessions_sweep".

  value : req/s with prompts resident in HBM (device tokens), CUDA events.
  e2e   : req/s through PrefillShareEngine.serve() with HOST prompts
          (pinned H2D of the token ids and D2H of the generated ids inside
          the timed region).
  roofline : the dominant kernel (decode GEMV, weight streaming) timed live
          with CUDA events on its launch stream; plus decode attention (K6)
          at the config-2 and config-4 (32k x 16 modules) shapes and the
          prefill (tcgen05) TFLOP/s.
  cpu_baseline : the fp32 CPU oracle on a bounded sample of the same
          workload, batched like the GPU arm (2 of 32 layers of a prefill and
          of one module's 32-row decode step, one LM head), scaled to req/s.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
Under torchrun each rank serves its own batch (weak scaling, no data-path
collective); timing is max over ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

PROMPT = 4096
MAX_NEW = 256
N_MOD = 4
METRIC = "multi-model agent req/s (8B-shape shared prefill + 4 decode modules, 4k prompt, 256 out)"


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": d["hbm_gbs"], "bf16": d["bf16_tflops"], "bf16_sus": d["bf16_tflops_sustained"],
                "src": "measured"}
    return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sus": 1400.0, "src": "fallback"}


# --------------------------------------------------------------- clocks ----

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows: list[list[str]] = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True,
                                     text=True, timeout=5).stdout.strip()
                if out:
                    self.rows.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------ CPU oracle ---

class CpuReference:
    """The fp32 CPU oracle (oracle/model.py, the reference path restated) on
    a bounded sample of the same workload, run the way a batched CPU server
    would run it, scaled to req/s. One sample():
      * prefill: 2 full-width layers of one 4096-token prompt (t_pre2);
      * decode: 2 full-width layers of ONE module's co-batched step over its
        n_sessions rows (weights read once per step for all rows; each row
        attends over its own session's 4095-token shared KV plus its own
        token: oracle.decode_layer_batched) (t_dec2), and the module's LM
        head over those rows (t_head, full 128256 vocab);
      * per serve: n_sessions x 16 x t_pre2 + 256 x 4 modules x
        (16 x t_dec2 + t_head).
    The extrapolation factors (x16 layers, x4 modules of identical shape,
    x256 steps) are stated in the sample text. Weights and caches are built
    once (__init__), outside the timed samples."""

    L = 2

    def __init__(self, n_sessions: int = 32):
        import torch
        from oracle.model import layer_forward, rope_cos_sin
        from paper_2602_12029_b200.model import LlamaConfig
        torch.manual_seed(0)
        self.full = full = LlamaConfig.llama8b()
        self.cfg = cfg = LlamaConfig(n_layers=self.L, d_model=full.d_model, n_heads=full.n_heads,
                                     n_kv_heads=full.n_kv_heads, ffn=full.ffn, vocab=full.vocab,
                                     rope_theta=full.rope_theta, max_pos=PROMPT + MAX_NEW)
        d, f, hd = cfg.d_model, cfg.ffn, cfg.head_dim
        r = lambda *s: torch.randn(*s) * 0.02  # noqa: E731

        def layer():
            return {"attn_norm": 1 + 0.1 * torch.randn(d), "wq": r(cfg.n_heads * hd, d),
                    "wk": r(cfg.n_kv_heads * hd, d), "wv": r(cfg.n_kv_heads * hd, d),
                    "wo": r(d, cfg.n_heads * hd), "mlp_norm": 1 + 0.1 * torch.randn(d),
                    "w_gate": r(f, d), "w_up": r(f, d), "w_down": r(d, f)}
        self.base_l = [layer() for _ in range(self.L)]
        self.mod_l = [layer() for _ in range(self.L)]
        self.head = r(full.vocab, d)
        self.cos, self.sin = rope_cos_sin(cfg.max_pos, hd, cfg.rope_theta)
        self.R = n_sessions
        self.x_pre = r(PROMPT - 1, d) * 50
        self.x_dec = r(n_sessions, d) * 50
        with torch.inference_mode():
            x, kvs = self.x_pre, []
            for lw in self.base_l:
                x, kv = layer_forward(cfg, lw, x, None, self.cos, self.sin)
                kvs.append(kv)
        # every row of the batch attends over its own session's shared KV in
        # its own memory (R x 2 layers x 33.5 MB; one prompt's values
        # replicated: the arithmetic and the bytes read are a real batch's)
        self.pasts = [(k.unsqueeze(0).repeat(n_sessions, 1, 1, 1), v.unsqueeze(0).repeat(n_sessions, 1, 1, 1))
                      for k, v in kvs]

    def sample(self) -> dict:
        import torch
        from oracle.model import decode_layer_batched, layer_forward
        cfg = self.cfg
        with torch.inference_mode():
            t0 = time.perf_counter()
            x = self.x_pre
            for lw in self.base_l:
                x, _ = layer_forward(cfg, lw, x, None, self.cos, self.sin)
            t_pre2 = time.perf_counter() - t0
            t0 = time.perf_counter()
            xs = self.x_dec
            for lw, (kp, vp) in zip(self.mod_l, self.pasts):
                xs, _ = decode_layer_batched(cfg, lw, xs, kp, vp, self.cos, self.sin)
            t_dec2 = time.perf_counter() - t0
            t0 = time.perf_counter()
            _ = xs @ self.head.T
            t_head = time.perf_counter() - t0
        S, lf = self.R, self.full.n_layers // self.L
        per_serve = S * lf * t_pre2 + MAX_NEW * N_MOD * (lf * t_dec2 + t_head)
        return {"value": S * N_MOD / per_serve, "unit": "req/s", "cores": torch.get_num_threads(), "kind": "port",
                "sample": (f"fp32 CPU oracle, batched like the GPU arm: 2 of 32 full-width layers of a 4096-token "
                           f"prefill ({t_pre2:.2f} s), 2 layers of one module's decode step over {S} co-batched "
                           f"rows ({t_dec2 * 1e3:.1f} ms), one module's LM head over {S} rows "
                           f"({t_head * 1e3:.1f} ms); scaled x{lf} layers, x{N_MOD} modules of the same shape, "
                           f"x{MAX_NEW} steps, x{S} prefills per serve of {S} sessions")}


# --------------------------------------------------------- kernel timing ---

def _time_launches(fn, n: int, graph: bool = True) -> float:
    """Average device time of one fn() launch sequence: n launches captured in
    a CUDA graph (no host launch overhead in the timing), replayed and timed
    with CUDA events on the capturing stream."""
    import torch
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    st.synchronize()
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(n):
                fn()
        run = g.replay
    else:
        def run():
            for _ in range(n):
                fn()
    with torch.cuda.stream(st):
        run()
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        run()
        b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / 1e3 / n


def gemv_roofline(eng, peaks) -> dict:
    """Dominant kernel: the grouped gate/up GEMV (4 modules x 235 MB weights
    per launch), timed back-to-back over the 32 layers' weights (working set
    7.5 GB >> L2)."""
    import torch
    from paper_2602_12029_b200 import _lib
    r = eng.runner
    lib, cfg, b = r.lib, eng.cfg, eng.batch
    s = torch.cuda.current_stream().cuda_stream
    it = [0]

    def launch():  # the engine's own dispatch: K5 (<= 8 rows/module) or K5-TC
        l = it[0] % cfg.n_layers
        it[0] += 1
        r._gemv(r.xn, cfg.d_model, r.p_wgu[l], r.h_wgu[l], 2 * cfg.ffn, 3, r.act,
                torch.cuda.current_stream().cuda_stream)
    dt = _time_launches(launch, 4 * cfg.n_layers)
    nbytes = b.n_mod * 2 * cfg.ffn * cfg.d_model * 2 + b.n_rows * (cfg.d_model + cfg.ffn) * 2
    gbs = nbytes / dt / 1e9
    # DRAM bytes per launch of this kernel at this shape from the committed
    # `ncu --set full` capture (tools/profile_kernels.py gemv <rows/module>)
    traffic, tsrc = None, None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        t = json.loads(tf.read_text()).get(f"gemv_gate_up_m{b.max_rpm}" + ("_tc" if r.use_tc_gemv else ""))
        if t:
            traffic, tsrc = t["dram_bytes"], t["source"]
    kname = "psk_gemv_tc (tcgen05" if r.use_tc_gemv else "psk_gemv (mma.sync"
    return {"bound": "hbm", "kernel": f"{kname}; gate/up, SiLU*mul epilogue)", "achieved": round(gbs, 1),
            "peak": peaks["hbm"], "unit": "GB/s", "frac": round(gbs / peaks["hbm"], 4),
            "traffic": traffic, "traffic_source": tsrc, "bytes_per_launch": nbytes,
            "us_per_launch": round(dt * 1e6, 2), "rows_per_module": b.max_rpm,
            "peak_source": peaks["src"],
            "peak_note": ("MEASURED_PEAKS hbm_gbs is a device copy (read+write); the pure-read "
                          "ceiling measured by tools/bw_probe.cu is ~7.05-7.25 TB/s, so frac > 1 "
                          "is possible for this read-only stream")}


def decode_attn_roofline(eng, peaks) -> dict:
    """K6 on the engine's live batch (shared 4095-token prefix, 4 modules),
    cycling the 32 layers (512 MiB of KV, > L2)."""
    import torch
    from paper_2602_12029_b200 import _lib
    r = eng.runner
    cfg, b = eng.cfg, eng.batch
    kvl = eng.kv.layout()
    s = torch.cuda.current_stream().cuda_stream
    b.t_priv_len.fill_(MAX_NEW - 1)  # state of the last decode step
    it = [0]

    def launch():
        l = it[0] % cfg.n_layers
        it[0] += 1
        _lib.check(r.lib.psk_decode_attn(b.c_ref(), r.q_rot.data_ptr(), cfg.n_heads, l, kvl,
                                         r.splits, r.ws.data_ptr(), r.attn.data_ptr(),
                                         torch.cuda.current_stream().cuda_stream))
    dt = _time_launches(launch, 4 * cfg.n_layers)
    shared = int(b.t_sess_len.sum().item())
    priv = int((b.t_priv_len + 1).sum().item())
    per_tok = 2 * cfg.n_kv_heads * cfg.head_dim * 2
    nbytes = (shared + priv) * per_tok + 2 * b.n_rows * cfg.n_heads * cfg.head_dim * 2
    gbs = nbytes / dt / 1e9
    return {"shape": f"{b.n_sess} session(s) x {shared // max(1, b.n_sess)} shared tokens, {b.n_rows} rows",
            "achieved": round(gbs, 1), "unit": "GB/s", "frac": round(gbs / peaks["hbm"], 4),
            "bytes_per_launch": nbytes, "us_per_launch": round(dt * 1e6, 2)}


def decode_attn_fanout(peaks, shared_tokens=32767, modules=16, sessions=1, priv=1, splits=None) -> dict:
    """K6 at a fan-out shape: `sessions` shared contexts of `shared_tokens`,
    each read by `modules` decode modules (4 query heads per KV head each)
    with `priv` private tokens per row, random KV / queries, 32 layers cycled
    (working set > L2). Default: the config-4 shape (32k x 16 modules)."""
    import torch
    from paper_2602_12029_b200 import _lib
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, KVCache, LlamaConfig,
                                             SessionSpec)
    cfg = LlamaConfig.llama8b(max_pos=shared_tokens + priv + 64)
    n_sh = (shared_tokens + 15) // 16
    n_pr = (priv + 15) // 16
    per_sess = n_sh + modules * n_pr
    kv = KVCache(cfg, sessions * per_sess)
    lib = _lib.load()
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(lib.psk_init_normal_bf16(kv.data.data_ptr(), kv.data.numel(), 99, 1.0, s))
    rows, sess = [], []
    for si in range(sessions):
        base = si * per_sess
        sess.append(SessionSpec(shared_len=shared_tokens, pages=list(range(base, base + n_sh))))
        rows += [DecodeRow(module=m, session=si, first_token=0,
                           pages=list(range(base + n_sh + m * n_pr, base + n_sh + (m + 1) * n_pr)))
                 for m in range(modules)]
    b = DecodeBatch(sess, rows, modules)
    b.t_priv_len.fill_(priv - 1)
    R = sessions * modules
    q = torch.randn(R, cfg.n_heads, cfg.head_dim, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    import ctypes
    from paper_2602_12029_b200.model import attn_splits
    # splits: None = fixed split count (one CTA per SM over the groups), 0 = stream-K
    ns = splits if splits is not None else attn_splits(
        per_sess, cfg.n_kv_heads * sessions, torch.cuda.get_device_properties(0).multi_processor_count)
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_decode_attn_workspace(b.c_ref(), cfg.n_kv_heads, ns, ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value // 4 + 1, dtype=torch.float32, device="cuda")
    it = [0]
    kvl = kv.layout()

    def launch():
        l = it[0] % cfg.n_layers
        it[0] += 1
        _lib.check(lib.psk_decode_attn(b.c_ref(), q.data_ptr(), cfg.n_heads, l, kvl, ns,
                                       ws.data_ptr(), out.data_ptr(),
                                       torch.cuda.current_stream().cuda_stream))
    dt = _time_launches(launch, 2 * cfg.n_layers)
    per_tok = 2 * cfg.n_kv_heads * cfg.head_dim * 2
    nbytes = sessions * (shared_tokens + modules * priv) * per_tok + 2 * R * cfg.n_heads * cfg.head_dim * 2
    gbs = nbytes / dt / 1e9
    del kv
    torch.cuda.empty_cache()
    return {"shape": f"{sessions} session(s) x {shared_tokens} shared tokens, {modules} modules, "
                     f"{priv} private tokens/row",
            "achieved": round(gbs, 1), "unit": "GB/s", "frac": round(gbs / peaks["hbm"], 4),
            "bytes_per_launch": nbytes, "us_per_launch": round(dt * 1e6, 2),
            "per_model_reread_bytes": sessions * modules * shared_tokens * per_tok}


def pool_ops(n_tokens: int = PROMPT, reps: int = 50) -> dict:
    """K7 through the BlockPool drop-in API (host query staging + kernel +
    result read-back per call, as the engine calls it) vs the CPU oracle pool
    (oracle/pool.py, the reference kvstore.py algorithm) on identical ops:
    insert of a fresh 4096-token prompt (256 blocks) and its full-hit lookup."""
    import numpy as np
    from oracle.pool import OraclePool
    from paper_2602_12029_b200.kvstore import SHARED_NS, BlockPool
    rng = np.random.default_rng(5)
    prompts = [rng.integers(0, 1 << 40, n_tokens, dtype=np.int64) for _ in range(reps)]
    cap = reps * (n_tokens // 16) + 16
    out = {"tokens": n_tokens, "blocks": n_tokens // 16}
    for name, pool in (("gpu", BlockPool(cap, 16)), ("cpu_oracle", OraclePool(cap, 16))):
        tup = [tuple(int(x) for x in p) for p in prompts] if name == "cpu_oracle" else prompts
        t0 = time.perf_counter()
        for i, p in enumerate(tup):
            pool.insert(SHARED_NS, p, i)
        t1 = time.perf_counter()
        for i, p in enumerate(tup):
            if name == "gpu":
                m, chain = pool.longest_prefix_match(SHARED_NS, p, reps + i)
                pool.release(chain)
            else:
                ids = pool.lookup(SHARED_NS, p, reps + i)
                pool.release(ids)
                m = len(ids) * 16
            assert m == n_tokens
        t2 = time.perf_counter()
        out[name] = {"insert_us": round((t1 - t0) / reps * 1e6, 1),
                     "lookup_hit_us": round((t2 - t1) / reps * 1e6, 1)}
    out["cpu_oracle"].update(cores=1, kind="port")
    return out


def kv_copy_roofline(eng, peaks, n_pages: int = PROMPT // 16 + 1) -> dict:
    """K8: move one 4k-token context's pages (257 x 2 MiB, all layers) inside
    the pool, as the same-process handoff does (transfer.copy_pages)."""
    import torch
    from paper_2602_12029_b200 import _lib
    kv = eng.kv
    P = kv.data.shape[0]
    src = torch.arange(0, n_pages, dtype=torch.int32, device="cuda")
    dst = torch.arange(P - n_pages, P, dtype=torch.int32, device="cuda")
    page_bytes = kv.data[0].numel() * 2
    lib = _lib.load()

    def launch():
        _lib.check(lib.psk_kv_copy_pages(kv.data.data_ptr(), kv.data.data_ptr(), src.data_ptr(),
                                         dst.data_ptr(), n_pages, page_bytes,
                                         torch.cuda.current_stream().cuda_stream))
    dt = _time_launches(launch, 8)
    nbytes = 2 * n_pages * page_bytes  # read + write
    gbs = nbytes / dt / 1e9
    return {"bound": "hbm", "pages": n_pages, "bytes_per_launch": nbytes, "us_per_launch": round(dt * 1e6, 2),
            "achieved": round(gbs, 1), "unit": "GB/s", "frac": round(gbs / peaks["hbm"], 4)}


def serve_point(cfg, mods, base, S: int, batches, device: int, steps: int = 2) -> dict:
    """req/s and p95 serve latency of an engine serving S sessions per step
    on the given weights (prompts resident in HBM is not needed: host
    prompts, the e2e path). One warm-up serve, then `steps` timed serves."""
    import numpy as np
    import torch
    from paper_2602_12029_b200.engine import PrefillShareEngine
    e = PrefillShareEngine(cfg, N_MOD, S, PROMPT, MAX_NEW, pool_pages=S * (PROMPT // 16 + 1) + 64,
                           device=device, modules=mods, base=base)
    e.capture()
    rng = np.random.default_rng(77 + S)
    prompts = [[rng.integers(0, cfg.vocab, PROMPT, dtype=np.int64) for _ in range(S)] for _ in range(steps + 1)]
    e.serve(prompts[0])
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    ev[0].record(st)
    for j in range(steps):
        e.serve(prompts[j + 1])
        ev[j + 1].record(st)
    ev[-1].synchronize()
    ts = [ev[j].elapsed_time(ev[j + 1]) / 1e3 for j in range(steps)]
    del e
    torch.cuda.empty_cache()
    return {"sessions": S, "value": round(S * N_MOD * steps / sum(ts), 4), "unit": "req/s",
            "p95_latency_ms": round(max(ts) * 1e3, 2)}


def agents_point(cfg, mods, base, rate: float = 8.0, duration: float = 20.0, rows: int = 64,
                 pool_pages: int = 7500) -> dict:
    """BASELINE configs 3 / 5 on one GPU: the reference's agent workload
    (workload.generate, ReAct, Poisson arrivals at `rate` sessions/s for
    `duration` s, seed 0) served in real time by serve.AgentServer in both
    modes on the same weights: per-request p95 E2E / TTFT under arrivals
    (metrics.py definitions, GPU-completion timestamps) next to the batch
    number. BASELINE: one prefill worker + pool per model; PREFILLSHARE: the
    frozen base module prefills for every model, sessions pinned to the
    least-queued of the per-worker pools (router.py:58-77), 7500 blocks per
    worker (config.py:39), 64 decode rows per model (max_batch)."""
    import torch
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.router import ServingMode
    from paper_2602_12029_b200.serve import AgentServer, summarize
    models = list(wl.DEFAULT_MODELS)
    sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=rate, duration_s=duration,
                                             seed=0))
    out = {"workload": f"configs[2]/[4] on 1 GPU: react, {rate:g} sessions/s for {duration:g} s, "
                       f"{len(sessions)} sessions, {sum(s.total_requests for s in sessions)} requests",
           "rows_per_model": rows, "pool_blocks_per_worker": pool_pages}
    for mode in (ServingMode.BASELINE, ServingMode.PREFILLSHARE):
        srv = AgentServer(cfg, models, mode, rows_per_module=rows, pool_pages_per_worker=pool_pages,
                          max_context=4096, max_output=256, modules=mods, base=base)
        recs = srv.run(sessions)
        sm = summarize(recs)
        out[mode.value] = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in sm.items()}
        del srv
        torch.cuda.empty_cache()
    b, p = out["baseline"], out["prefillshare"]
    if b.get("req_per_s") and p.get("req_per_s"):
        out["req_per_s_ratio"] = round(p["req_per_s"] / b["req_per_s"], 3)
        out["p95_e2e_ratio"] = round(b["p95_e2e_ms"] / p["p95_e2e_ms"], 3)
    return out


def pd_split_point(world: int, rank: int, local: int, ctrl, duration: float = 10.0, rows: int = 32,
                   pool_pages: int = 7500, cfg=None, place=None, max_context: int = 4096,
                   max_output: int = 256) -> dict | None:
    """BASELINE configs 3 / 5 on the N-GPU prefill/decode split
    (north_star: "2/4/8-GPU prefill/decode splits"): the reference fleet's
    4 logical prefill workers (own 7500-block pools) on P = max(1, N/4)
    prefill GPUs, the 4 models' decode workers replicated over the other
    N - P GPUs (router.Placement.split(replicate=True): 2P + 6D uses all six
    decode GPUs), disagg.DisaggServer serving workload.generate (ReAct,
    Poisson arrivals at 4 x N sessions/s for `duration` s: the offered load
    grows with the fleet) in real time, BASELINE then PREFILLSHARE on the
    same weights. Per mode: req/s, p95 E2E / TTFT (GPU completion times),
    prefix hit ratio, and the cross-GPU KV handoff volume and GB/s (packed
    per peer pair, NCCL P2P over NVLink; sender-side pack + transfer time).
    Every rank runs it; rank 0 returns the dict."""
    import torch
    import torch.distributed as dist
    from paper_2602_12029_b200 import workload as wl
    from paper_2602_12029_b200.disagg import (Coordinator, DisaggServer, GpuDecodeBackend, GpuPrefillBackend,
                                              summarize)
    from paper_2602_12029_b200.model import LlamaConfig, ModuleWeights
    from paper_2602_12029_b200.router import Placement, Router, ServingMode
    models = list(wl.DEFAULT_MODELS)
    M = len(models)
    if place is None:
        P = max(1, world // 4)
        place = Placement.split(M, list(range(P)), list(range(P, world)), M, replicate=True)
    cfg = cfg or LlamaConfig.llama8b(max_pos=max_context + 512)
    ctx_pages_per_row = max_context // 16 + 4
    mine_p = [w for w, r in enumerate(place.prefill_gpus) if r == rank]
    mine_d = place.decode_models_on(rank)
    rate = 4.0 * world
    sessions = wl.generate(wl.WorkloadConfig(pattern="react", arrival_rate_per_s=rate, duration_s=duration, seed=0))
    out = {"workload": f"configs[2]/[4]: react, {rate:g} sessions/s for {duration:g} s, {len(sessions)} sessions, "
                       f"{sum(s.total_requests for s in sessions)} requests",
           "placement": {"prefill_gpus": list(place.prefill_gpus),
                         "decode_replicas": [list(place.replicas(m)) for m in range(M)]},
           "rows_per_model_replica": rows, "pool_blocks_per_worker": pool_pages}
    for mode in (ServingMode.BASELINE, ServingMode.PREFILLSHARE):
        base = (ModuleWeights(cfg, 99, with_head=False, device=local)
                if mine_p and mode is ServingMode.PREFILLSHARE else None)
        need = set(mine_d) | (set(mine_p) if mode is ServingMode.BASELINE else set())
        mods = {m: ModuleWeights(cfg, 100 + m, device=local) for m in sorted(need)}
        prefill = {w: GpuPrefillBackend(cfg, base if base is not None else mods[w], pool_pages, max_context, 256,
                                        local) for w in mine_p}
        decode = (GpuDecodeBackend(cfg, {m: mods[m] for m in mine_d}, rows,
                                   ctx_pages=len(mine_d) * rows * ctx_pages_per_row, max_context=max_context,
                                   max_output=max_output, device=local) if mine_d else None)
        srv = DisaggServer(place, models, mode, prefill, decode, rows, ctrl_group=ctrl)
        coord = Coordinator(sessions, models, Router(mode, models), place, steps_per_round=8) if rank == 0 else None
        torch.cuda.synchronize()
        dist.barrier(group=ctrl)
        recs = srv.run(coord)
        torch.cuda.synchronize()
        hs = [None] * world if rank == 0 else None
        dist.gather_object(srv.handoff_stats(), hs, dst=0, group=ctrl)
        if rank == 0:
            sm = {k: (round(v, 4) if isinstance(v, float) else v) for k, v in summarize(recs).items()}
            nb = sum(h["bytes"] for h in hs)
            sec = max(h["seconds"] for h in hs)
            sm["handoff"] = {"bytes": nb, "gbs_per_sender": [round(h["gbs"], 1) if h["gbs"] else None for h in hs],
                             "aggregate_gbs": round(nb / sec / 1e9, 1) if sec > 0 else None}
            out[mode.value] = sm
        del srv, prefill, decode, mods, base
        torch.cuda.empty_cache()
    if rank != 0:
        return None
    b, p = out["baseline"], out["prefillshare"]
    if b.get("req_per_s") and p.get("req_per_s"):
        out["req_per_s_ratio"] = round(p["req_per_s"] / b["req_per_s"], 3)
        out["p95_e2e_ratio"] = round(b["p95_e2e_ms"] / p["p95_e2e_ms"], 3)
    return out


def tinylm_point(n_prompts: int = 32, n: int = 255, ratio: float = 0.5, reps: int = 5) -> dict:
    """The reference's own TinyLM at its DEFAULT_MODEL (model.ts:26-31: 4
    layers, width 128, 4 heads, 256 context; vocab 64): one evaluateSharing
    call (evaluate.ts:21-50: base cache of n prompts, slice at m = ceil(r n),
    decode module's forward of the tails, greedy predictions) through the
    public API (host prompts in, host predictions out), GPU (psk_tiny_forward,
    fp32) vs the CPU oracle restatement on the same call (torch fp32, all host
    threads). Wall time per call, median of `reps`."""
    import torch

    import oracle.tinylm as O
    from paper_2602_12029_b200 import tinylm as G
    shape = (4, 128, 4, 256, 64)
    pool = G.TinyKVPool(G.TinyConfig(*shape), n_prompts * 2 * (n // 16 + 2) + 16)
    gb, gd = G.TinyLM.init(G.TinyConfig(*shape), 1, pool=pool), G.TinyLM.init(G.TinyConfig(*shape), 2, pool=pool)
    ob, od = O.TinyLM.init(O.TinyConfig(*shape), 1), O.TinyLM.init(O.TinyConfig(*shape), 2)
    r = O.Rng(7)
    prompts = [[r.int(64) for _ in range(n)] for _ in range(n_prompts)]

    def gpu_call():
        pool.next = 0  # the call's pages are reused (same shapes every rep)
        pool.filled[:] = 0
        return G.sharing_predictions(gd, gb, ratio, prompts)

    gpu_call()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = gpu_call()
        ts.append(time.perf_counter() - t0)
    t0 = time.perf_counter()
    want = O.evaluate_sharing_predictions(od, ob, ratio, prompts)
    t_cpu = time.perf_counter() - t0
    g_ms = statistics.median(ts) * 1e3
    return {"workload": f"evaluateSharing at r={ratio}: {n_prompts} prompts x {n} tokens, DEFAULT_MODEL",
            "gpu_ms_per_call": round(g_ms, 2), "cpu_oracle_ms_per_call": round(t_cpu * 1e3, 1),
            "cpu_threads": torch.get_num_threads(), "predictions_match_oracle": got == want}


def prefill_roofline(eng, peaks) -> dict:
    import torch
    T = PROMPT
    toks = torch.randint(0, eng.cfg.vocab, (T,), device="cuda", dtype=torch.int64)
    pt = torch.arange(eng.pool_pages - (T + 15) // 16, eng.pool_pages, dtype=torch.int32, device="cuda")
    dt = _time_launches(lambda: eng.prefill.run(toks, 0, pt), 3)
    fl = eng.prefill.flops(T)
    tf = fl / dt / 1e12
    return {"bound": "tensor", "tokens": T, "achieved": round(tf, 1), "unit": "TFLOP/s",
            "peak": peaks["bf16_sus"], "frac": round(tf / peaks["bf16_sus"], 4),
            "ms_per_prefill": round(dt * 1e3, 2)}


# ----------------------------------------------------------------- main ----

def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sessions", type=int, default=32, help="concurrent sessions per serve() batch")
    ap.add_argument("--no-extras", action="store_true", help="skip kernel rooflines / cpu baseline")
    a = ap.parse_args()
    a.warmup = max(3, a.warmup)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    config = {"workload": "configs[1]: Llama-3.1-8B-shape shared prefill + 4 decode modules, "
                          "4k-token shared prompt, 256 output tokens",
              "model": "llama-3.1-8b-shape (random init)", "sessions_per_step": a.sessions,
              "prompt_tokens": PROMPT, "output_tokens": MAX_NEW, "decode_modules": N_MOD,
              "l2": "inputs larger than L2 (60 GB of decode weights streamed per token step)"}

    if a.impl == "reference":
        if rank != 0:
            return
        ref = CpuReference(a.sessions)
        samples = [ref.sample() for _ in range(a.warmup + a.steps)][a.warmup:]
        v = statistics.median(s["value"] for s in samples)
        cb = dict(samples[-1])
        cb["value"] = v
        print(json.dumps({"metric": METRIC, "value": v, "unit": "req/s", "impl": "reference",
                          "n_gpus": a.gpus, "steps": a.steps, "warmup": a.warmup,
                          "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                          "dtype": "f32", "data": "synthetic", "config": config, "cpu_baseline": cb,
                          "e2e": {"value": v, "unit": "req/s", "h2d_bytes_per_step": 0,
                                  "d2h_bytes_per_step": 0}}))
        return

    import numpy as np
    import torch
    import torch.distributed as dist
    torch.cuda.set_device(local)
    ctrl = None
    if world > 1:
        import datetime
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # host control plane of the P/D split (and a long-timeout barrier
        # while rank 0 runs the single-GPU extras)
        ctrl = dist.new_group(backend="gloo", timeout=datetime.timedelta(hours=1))
    from paper_2602_12029_b200.engine import PrefillShareEngine
    from paper_2602_12029_b200.model import LlamaConfig
    peaks = _peaks()
    cfg = LlamaConfig.llama8b(max_pos=PROMPT + MAX_NEW + 64)
    S = a.sessions
    steps_total = a.warmup + 2 * a.steps
    pool_pages = max(2048, 3 * S * (PROMPT // 16 + 1))  # LRU-evicts older prompts
    eng = PrefillShareEngine(cfg, N_MOD, S, PROMPT, MAX_NEW, pool_pages=pool_pages,
                             seed=1000 * rank + 1, device=local)
    rng = np.random.default_rng(1234 + rank)
    batches = [[rng.integers(0, cfg.vocab, PROMPT, dtype=np.int64) for _ in range(S)]
               for _ in range(steps_total)]
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    eng.capture()
    for i in range(a.warmup):
        eng.serve(batches[i])
    # ---- value: prompts resident in HBM
    dev_batches = []
    for j in range(a.steps):
        t = torch.zeros(S, PROMPT, dtype=torch.int64, device="cuda")
        for s in range(S):
            t[s] = torch.from_numpy(batches[a.warmup + j][s]).cuda()
        dev_batches.append(t)
    st = torch.cuda.current_stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    barrier()
    with ClockSampler(local) as clk:
        ev[0].record(st)
        phases = []
        for j in range(a.steps):
            eng.serve(batches[a.warmup + j], device_tokens=dev_batches[j])
            ev[j + 1].record(st)
            phases.append(eng.last_phase_ms)
        ev[-1].synchronize()
    barrier()
    step_s = [ev[j].elapsed_time(ev[j + 1]) / 1e3 for j in range(a.steps)]
    t_val = max_over_ranks(sum(step_s))
    # ---- e2e: host prompts through the public API
    ev2 = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    barrier()
    ev2[0].record(st)
    for j in range(a.steps):
        eng.serve(batches[a.warmup + a.steps + j])
        ev2[j + 1].record(st)
    ev2[-1].synchronize()
    barrier()
    e2e_steps = [ev2[j].elapsed_time(ev2[j + 1]) / 1e3 for j in range(a.steps)]
    t_e2e = max_over_ranks(sum(e2e_steps))
    reqs = S * N_MOD * a.steps * world
    value = reqs / t_val
    e2e = reqs / t_e2e
    # per-request latency = its serve() duration (all modules finish together)
    lat = sorted(step_s)
    p95 = lat[min(len(lat) - 1, max(0, int(np.ceil(0.95 * len(lat))) - 1))]
    out = {"metric": METRIC, "value": round(value, 4), "unit": "req/s", "n_gpus": world,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": round(t_val / a.steps * 1e3, 2),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
           "data": "synthetic (random-init weights, random prompt ids)", "config": config,
           "p95_latency_ms": round(p95 * 1e3, 2),
           "e2e": {"value": round(e2e, 4), "unit": "req/s", "h2d_bytes_per_step": S * PROMPT * 8,
                   "d2h_bytes_per_step": S * N_MOD * MAX_NEW * 4,
                   "p95_latency_ms": round(sorted(e2e_steps)[-1] * 1e3, 2)},
           "gpu_launches": eng.launches_per_serve(S, S) * a.steps,
           # device time per serve: prefill phase (pool ops + grouped prefills) / decode phase
           "serve_phases_ms": {k: round(sum(p[k] for p in phases) / len(phases), 1) for k in ("prefill", "decode")},
           "clocks": clk.summary()}
    if not a.no_extras and rank == 0:
        out["roofline"] = gemv_roofline(eng, peaks)
        out["decode_attn"] = decode_attn_roofline(eng, peaks)
        out["prefill"] = prefill_roofline(eng, peaks)
        out["kv_copy"] = kv_copy_roofline(eng, peaks)
        step_bytes = eng.runner.weight_bytes_per_step
        out["decode_step"] = {"weight_bytes": step_bytes,
                              "ms_per_token_step": round(out["serve_phases_ms"]["decode"] / MAX_NEW, 3)}
        # throughput / latency at other batch sizes, same weights (the KV
        # pool of the main engine is freed first)
        mods, base = eng.mods, eng.base
        del eng
        torch.cuda.empty_cache()
        if world == 1:  # single-GPU serving points (N > 1: the P/D split below)
            out["sessions_sweep"] = [serve_point(cfg, mods, base, n, batches, local)
                                     for n in (1, 8, 64) if n != S]
            out["agents"] = agents_point(cfg, mods, base)
        del mods, base
        torch.cuda.empty_cache()
        out["decode_attn_fanout_32k_x16"] = decode_attn_fanout(peaks)
        out["pool"] = pool_ops()
        out["tinylm"] = tinylm_point()
        if world == 1:
            ref = CpuReference(S)
            ref.sample()  # warm-up
            out["cpu_baseline"] = ref.sample()
            del ref
    if world > 1 and not a.no_extras:
        # every rank: the prefill/decode split on this node's N GPUs
        if "eng" in locals():
            del eng
        torch.cuda.empty_cache()
        dist.barrier(group=ctrl)
        pd = pd_split_point(world, rank, local, ctrl)
        if rank == 0:
            out["pd_split"] = pd
    if rank == 0:
        print(json.dumps(out))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
