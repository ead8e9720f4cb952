"""Time the 8B-shape prefill module (4096-token prompt, 32 layers) and its
causal attention alone (K3, per layer), CUDA-graph replay, CUDA events.
PSK_PREFILL_TC1=1 selects the previous single-tile tcgen05 kernel.

    python tools/bench_prefill.py [T] [quick]   (quick: whole-prefill line only)
"""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_12029_b200 import _lib  # noqa: E402
from paper_2602_12029_b200.model import KVCache, LlamaConfig, ModuleWeights, PrefillRunner  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
import os  # noqa: E402
if os.environ.get("PSK_SEED") is not None:  # fixed prompt / queries (A/B runs)
    torch.manual_seed(int(os.environ["PSK_SEED"]))
cfg = LlamaConfig.llama8b(max_pos=T + 64)
base = ModuleWeights(cfg, 3, with_head=False)
kv = KVCache(cfg, T // 16 + 8)
pre = PrefillRunner(cfg, base, kv, max_tokens=T)
toks = torch.randint(0, cfg.vocab, (T,), device="cuda")
pt = torch.arange(T // 16 + 1, dtype=torch.int32, device="cuda")
if "attnonly" in sys.argv[2:]:  # K3 alone: fill the KV once, no whole-prefill timing (power state)
    pre.run(toks, 0, pt)
    torch.cuda.synchronize()
    dt = None
else:
    dt = bench._time_launches(lambda: pre.run(toks, 0, pt), 3)
    fl = pre.flops(T)
    print(f"prefill T={T}: {dt * 1e3:.2f} ms  {fl / dt / 1e12:.1f} TFLOP/s")
if "quick" in sys.argv[2:]:
    sys.exit(0)
if "batch" in sys.argv[2:]:  # G sequences of T tokens: G x run() vs one run_batch()
    for G in (2, 4):
        kvb = KVCache(cfg, G * (T // 16 + 1) + 8)
        preb = PrefillRunner(cfg, base, kvb, max_tokens=G * T)
        seqs = [(torch.randint(0, cfg.vocab, (T,), device="cuda"), 0,
                 list(range(g * (T // 16 + 1), (g + 1) * (T // 16 + 1)))) for g in range(G)]
        pts = [torch.tensor(p_, dtype=torch.int32, device="cuda") for _, _, p_ in seqs]

        def each():
            for (t_, p0, _), pt_ in zip(seqs, pts):
                preb.run(t_, p0, pt_)
        de = bench._time_launches(each, 3, graph=False)
        db = bench._time_launches(lambda: preb.run_batch(seqs), 3, graph=False)
        print(f"G={G} x T={T}: {G} x run {de * 1e3:.2f} ms | run_batch {db * 1e3:.2f} ms "
              f"({de / db:.3f}x)", flush=True)
    sys.exit(0)
lib = _lib.load()
q = torch.randn(T, cfg.n_heads, cfg.head_dim, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
kvl = kv.layout()
it = [0]


def attn():
    _lib.check(lib.psk_prefill_attn(q.data_ptr(), T, 0, cfg.n_heads, kvl, it[0] % cfg.n_layers, pt.data_ptr(),
                                    out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    it[0] += 1


import threading  # noqa: E402
clocks, stop = [], threading.Event()


def _poll():
    try:
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        while not stop.is_set():
            clocks.append(pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM))
            stop.wait(0.005)
    except Exception:  # noqa: BLE001
        pass


th = threading.Thread(target=_poll, daemon=True)
th.start()
reps = 5 if "attnonly" in sys.argv[2:] else 1
das = [bench._time_launches(attn, 64 if reps > 1 else 16) for _ in range(reps)]
stop.set()
th.join()
da = min(das)
afl = 4 * cfg.n_heads * cfg.head_dim * (T * (T + 1) / 2)  # QK^T + PV over the causal triangle
clk = sorted(clocks)[len(clocks) // 2] if clocks else -1  # median SM clock while timing
print(f"prefill attention T={T}: {da * 1e6:.1f} us/layer  {afl / da / 1e12:.1f} TFLOP/s (causal flops) "
      f"sm_clock_median={clk} MHz runs={[round(x * 1e6, 1) for x in das]}")
if "attn" in sys.argv[2:] or "attnonly" in sys.argv[2:]:
    sys.exit(0)

# in-situ ablation: prefill with one launch kind replaced by a no-op
kinds = {"gemm": ["psk_gemm", "psk_gemm_qkv_rope_kv"], "attention": ["psk_prefill_attn"],
         "rmsnorm": ["psk_rmsnorm_rows"], "embed": ["psk_embed_tokens"]}
for name, fns in kinds.items():
    saved = {f: getattr(lib, f) for f in fns}
    for f in fns:
        setattr(lib, f, lambda *a: 0)
    t = bench._time_launches(lambda: pre.run(toks, 0, pt), 3)
    for f, fn in saved.items():
        setattr(lib, f, fn)
    print(f"  without {name:10s} {t * 1e3:8.2f} ms -> in-situ {(dt - t) * 1e3:7.2f} ms")

# each GEMM shape alone (weights of all layers cycled)
A = torch.randn(T, 14336, device="cuda").to(torch.bfloat16)
shapes = {"qkv": (cfg.qkv_dim, 4096, base.wqkv), "o": (4096, 4096, base.wo), "gate_up": (2 * cfg.ffn, 4096, base.wgu),
          "down": (4096, cfg.ffn, base.wdown)}
for name, (N, K, ws) in shapes.items():
    o = torch.empty(T, N, dtype=torch.bfloat16, device="cuda")
    it2 = [0]

    def g():
        _lib.check(lib.psk_gemm(A.data_ptr(), ws[it2[0] % cfg.n_layers].data_ptr(), T, N, K, 0, o.data_ptr(), N,
                                torch.cuda.current_stream().cuda_stream))
        it2[0] += 1
    dg = bench._time_launches(g, 16)
    print(f"  gemm {name:8s} M={T} N={N:6d} K={K:6d}: {dg * 1e6:8.1f} us {2 * T * N * K / dg / 1e12:7.1f} TFLOP/s")
