"""In-situ cost of each kernel kind inside the captured decode step: the
step graph is re-captured with one kind of launch replaced by a no-op and
timed against the full step (numerics of the ablated graphs are garbage;
timing only). 8B shape, 4 modules x S sessions.

    python tools/step_ablation.py [S]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 8
P, NEW = 4096, 256
cfg = LlamaConfig.llama8b(max_pos=P + NEW + 16)
eng = PrefillShareEngine(cfg, n_modules=4, max_sessions=S, max_prompt=P, max_new=NEW,
                         pool_pages=S * (P // 16 + 1) + 64, seed=0)
rng = np.random.default_rng(0)
eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64) for _ in range(S)])
r = eng.runner
lib = r.lib


def time_step(n=40):
    r.b.t_priv_len.fill_(NEW // 2)  # mid-generation state, held fixed
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        r._step(st.cuda_stream)
        st.synchronize()
        with torch.cuda.graph(g, stream=st):
            for _ in range(4):
                r._step(st.cuda_stream)
        g.replay()
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(n // 4):
            g.replay()
        b.record(st)
    b.synchronize()
    return a.elapsed_time(b) / n * 1e3  # us per step


kinds = {"rmsnorm": ["psk_rmsnorm_rows"], "rope_append": ["psk_rope_append"], "attention": ["psk_decode_attn"],
         "gemv": ["psk_gemv", "psk_gemv_tc"], "qkv+rope fused": ["psk_gemv_tc_qkv_rope"],
         "embed+argmax": ["psk_embed_rows", "psk_argmax_advance"]}
full = time_step()
print(f"S={S}: full step {full:9.1f} us (fused QKV epilogue: {r.fused_qkv})", flush=True)
if "quick" in sys.argv[2:]:
    sys.exit(0)
for name, fns in kinds.items():
    saved = {f: getattr(lib, f) for f in fns}
    for f in fns:
        setattr(lib, f, lambda *a: 0)
    t = time_step()
    for f, fn in saved.items():
        setattr(lib, f, fn)
    print(f"  without {name:14s} {t:9.1f} us  -> in-situ cost {full - t:8.1f} us/step")

# each GEMV kind alone (the runner's dispatch no-op'ed for one (N, K) shape)
d, f, v = cfg.d_model, cfg.ffn, cfg.vocab
gemv_kinds = {"gemv qkv": (cfg.qkv_dim, d), "gemv o": (d, cfg.n_heads * cfg.head_dim), "gemv gate_up": (2 * f, d),
              "gemv down": (d, f), "gemv head": (v, d)}
orig = r._gemv
for name, (N0, K0) in gemv_kinds.items():
    def filt(x, K, p_dev, p_host, N, epi, out, s, N0=N0, K0=K0):
        if (N, K) != (N0, K0):
            orig(x, K, p_dev, p_host, N, epi, out, s)
    r._gemv = filt
    t = time_step()
    r._gemv = orig
    print(f"  without {name:14s} {t:9.1f} us  -> in-situ cost {full - t:8.1f} us/step", flush=True)
