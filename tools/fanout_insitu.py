"""K6 fan-out in situ at the config-4 shape: one 32767-token shared context
read by 16 decode modules (64 query rows per KV head) inside the real
graph-captured decode step, PDL-chained between the QKV GEMV (+RoPE/append)
and the o-proj GEMV as in serving. 8B-width modules truncated to L layers
(16 x 8B modules do not fit one GPU; per-layer attention work is unchanged
by the truncation). In-situ attention cost = step time - step time with
psk_decode_attn replaced by a no-op, per layer; bytes = the shared KV read
once + the rows' private KV + q / out, as bench.decode_attn_fanout.

    python tools/fanout_insitu.py [L] [modules] [shared_tokens]
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2602_12029_b200.engine import PrefillShareEngine  # noqa: E402
from paper_2602_12029_b200.model import LlamaConfig  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
MODS = int(sys.argv[2]) if len(sys.argv) > 2 else 16
P = int(sys.argv[3]) if len(sys.argv) > 3 else 32768
NEW = 16
cfg = LlamaConfig.llama8b(n_layers=L, max_pos=P + NEW + 16)
eng = PrefillShareEngine(cfg, n_modules=MODS, max_sessions=1, max_prompt=P, max_new=NEW,
                         pool_pages=P // 16 + 64, seed=0, prefill_group=1)
rng = np.random.default_rng(0)
eng.serve([rng.integers(0, cfg.vocab, P, dtype=np.int64)])
r = eng.runner
lib = r.lib
PRIV = NEW // 2


def time_step(n=64):
    r.b.t_priv_len.fill_(PRIV)  # mid-generation state, held fixed
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


res = []
for rep in range(3):
    full = time_step()
    saved = lib.psk_decode_attn
    lib.psk_decode_attn = lambda *a: 0
    wo = time_step()
    lib.psk_decode_attn = saved
    res.append((full, wo))
full = min(x[0] for x in res)
wo = min(x[1] for x in res)
per_layer = (full - wo) / L
shared = P - 1  # the decode modules process the last prompt token themselves
per_tok = 2 * cfg.n_kv_heads * cfg.head_dim * 2
nbytes = (shared + MODS * (PRIV + 1)) * per_tok + 2 * MODS * cfg.n_heads * cfg.head_dim * 2
peak = bench._peaks()["hbm"]
alone = bench.decode_attn_fanout(bench._peaks(), shared_tokens=shared, modules=MODS)
print(json.dumps({"shape": f"1 session x {shared} shared tokens, {MODS} modules, {PRIV + 1} private tokens/row",
                  "layers": L, "step_us": round(full, 1), "step_without_attention_us": round(wo, 1),
                  "insitu_us_per_layer": round(per_layer, 2), "bytes_per_layer": nbytes,
                  "insitu_gbs": round(nbytes / per_layer / 1e3, 1), "insitu_frac": round(nbytes / per_layer / 1e3 / peak, 4),
                  "alone_us": alone["us_per_launch"], "alone_frac": alone["frac"], "runs": res}))
