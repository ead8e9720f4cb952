"""Time the 8B-shape prefill module (4096-token prompt, 32 layers) and its
causal attention alone (K3, per layer), CUDA-graph replay, CUDA events.
PSK_PREFILL_TC1=1 selects the previous single-tile tcgen05 kernel.

    python tools/bench_prefill.py [T]
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
cfg = LlamaConfig.llama8b(max_pos=T + 64)
base = ModuleWeights(cfg, 3, with_head=False)
kv = KVCache(cfg, T // 16 + 8)
pre = PrefillRunner(cfg, base, kv, max_tokens=T)
toks = torch.randint(0, cfg.vocab, (T,), device="cuda")
pt = torch.arange(T // 16 + 1, dtype=torch.int32, device="cuda")
dt = bench._time_launches(lambda: pre.run(toks, 0, pt), 3)
fl = pre.flops(T)
print(f"prefill T={T}: {dt * 1e3:.2f} ms  {fl / dt / 1e12:.1f} TFLOP/s")
lib = _lib.load()
q = torch.randn(T, cfg.n_heads, cfg.head_dim, device="cuda").to(torch.bfloat16)
out = torch.empty_like(q)
kvl = kv.layout()
it = [0]


def attn():
    _lib.check(lib.psk_prefill_attn(q.data_ptr(), T, 0, cfg.n_heads, kvl, it[0] % cfg.n_layers, pt.data_ptr(),
                                    out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    it[0] += 1


da = bench._time_launches(attn, 16)
afl = 4 * cfg.n_heads * cfg.head_dim * (T * (T + 1) / 2)  # QK^T + PV over the causal triangle
print(f"prefill attention T={T}: {da * 1e6:.1f} us/layer  {afl / da / 1e12:.1f} TFLOP/s (causal flops)")
