"""K3 (prefill attention) and K6 (decode attention) at their full benchmarked
lengths, directly against a torch fp32 reference on identical bf16 inputs.

K3: 4096-token causal prefill at pos0 = 0, a partial prefill after a cached
prefix (pos0 = 2048), both through the single-sequence ping-pong kernel
(psk_prefill_attn: 16+ q-blocks, lazy O rescale over long key ranges), and
the batched kernel (psk_prefill_attn_batch) on stacked sequences of mixed
length (incl. one 4096-token item) with scattered page tables.
Tolerance: |out - ref| <= 2e-2 * max|ref| + 2e-3 per (token, head) row
block (bf16 P in the PV MMA, bf16 output, fp32 accumulation).

K6: the config-4 fan-out shape, 32767 shared tokens x 16 decode modules
(64 query rows per KV head -> the tcgen05 fan-out kernel), ragged private
suffixes, the engine's own split count, and 4095 x 4 modules x 32 sessions
(the bench's all-heads kernel). Same tolerance.
"""

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
RTOL, ATOL = 2e-2, 2e-3


def _cfg(n_layers=2, max_pos=40000):
    from paper_2602_12029_b200.model import LlamaConfig
    return LlamaConfig(n_layers=n_layers, d_model=4096, n_heads=32, n_kv_heads=8, ffn=256, vocab=64,
                       rope_theta=5e5, max_pos=max_pos)


def _gather(kv, pages, layer, n):
    """[n_kv, n, hd] K and V (bf16 on device) of positions [0, n)."""
    pv = kv.page_view()
    idx = torch.as_tensor(pages[:(n + 15) // 16], dtype=torch.long, device=kv.data.device)
    blk = pv[idx, layer]
    kvh = blk.permute(1, 2, 0, 3, 4).reshape(2, blk.shape[2], -1, blk.shape[-1])[:, :, :n]
    return kvh[0], kvh[1]


def _ref_prefill(q, K, V, pos0):
    """q [T, H, hd] bf16; K/V [n_kv, pos0+T, hd]. fp32 causal GQA attention."""
    T, H, hd = q.shape
    Hk = K.shape[0]
    grp = H // Hk
    out = torch.empty(T, H, hd, device=q.device)
    qpos = pos0 + torch.arange(T, device=q.device)
    mask = torch.arange(K.shape[1], device=q.device)[None, :] <= qpos[:, None]
    for g in range(Hk):
        Kg, Vg = K[g].float(), V[g].float()
        for h in range(g * grp, (g + 1) * grp):
            sc = (q[:, h].float() @ Kg.T) / np.sqrt(hd)
            sc = sc.masked_fill(~mask, float("-inf"))
            out[:, h] = torch.softmax(sc, -1) @ Vg
    return out


def _check(got, ref, what):
    err = (got.float() - ref).abs()
    scale = ref.abs().max().item()
    worst = err.max().item()
    assert worst <= RTOL * scale + ATOL, f"{what}: max err {worst} (scale {scale})"


@pytest.mark.parametrize("T,pos0", [(4096, 0), (2048, 2048), (1000, 3100)])
def test_k3_single_sequence_full_length(T, pos0):
    from paper_2602_12029_b200 import _lib
    from paper_2602_12029_b200.model import KVCache
    cfg = _cfg(max_pos=8192)
    n = pos0 + T
    n_pages = (n + 15) // 16
    rng = np.random.default_rng(T + pos0)
    pages = rng.permutation(n_pages + 7)[:n_pages].tolist()
    kv = KVCache(cfg, n_pages + 7)
    g = torch.Generator(device="cuda").manual_seed(3)
    kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
    q = torch.randn(T, cfg.n_heads, cfg.head_dim, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((T, cfg.n_heads * cfg.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    layer = 1
    pt = torch.tensor(pages, dtype=torch.int32, device="cuda")
    lib = _lib.load()
    _lib.check(lib.psk_prefill_attn(q.data_ptr(), T, pos0, cfg.n_heads, kv.layout(), layer, pt.data_ptr(),
                                    out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    K, V = _gather(kv, pages, layer, n)
    ref = _ref_prefill(q, K, V, pos0)
    _check(out.view(T, cfg.n_heads, cfg.head_dim), ref, f"K3 T={T} pos0={pos0}")


def test_k3_batched_items_mixed_lengths():
    """Stacked sequences (one 4096-token prefill, partial prefills after cached
    prefixes, tails ending mid-page, a 1-token item) through the batched
    kernel's (sequence, q-block, KV head) work items."""
    from paper_2602_12029_b200 import _lib
    from paper_2602_12029_b200.model import KVCache, batch_plan
    cfg = _cfg(max_pos=8192)
    specs = [(0, 4096), (2048, 300), (16, 1), (1500, 77), (0, 640)]  # (pos0, new tokens)
    rng = np.random.default_rng(9)
    total_pages = sum((p + n + 15) // 16 for p, n in specs)
    perm = rng.permutation(total_pages + 5).tolist()
    tables = [[perm.pop() for _ in range((p + n + 15) // 16)] for p, n in specs]
    kv = KVCache(cfg, total_pages + 5)
    g = torch.Generator(device="cuda").manual_seed(4)
    kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
    T = sum(n for _, n in specs)
    q = torch.randn(T, cfg.n_heads, cfg.head_dim, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full((T, cfg.n_heads * cfg.head_dim), float("nan"), dtype=torch.bfloat16, device="cuda")
    plan, n_items = batch_plan(cfg, [(n, p, pt) for (p, n), pt in zip(specs, tables)])
    dplan = torch.from_numpy(plan).cuda()
    ni = 8 * n_items
    layer = 0
    lib = _lib.load()
    _lib.check(lib.psk_prefill_attn_batch(q.data_ptr(), n_items, dplan.data_ptr(), cfg.n_heads, kv.layout(),
                                          layer, dplan.data_ptr() + 4 * (ni + 2 * T), out.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    off = 0
    for (p0, n), pt in zip(specs, tables):
        K, V = _gather(kv, pt, layer, p0 + n)
        ref = _ref_prefill(q[off:off + n], K, V, p0)
        _check(out[off:off + n].view(n, cfg.n_heads, cfg.head_dim), ref, f"K3 batch item pos0={p0} T={n}")
        off += n


def _k6_case(sess_lens, mods_per_sess, priv_lens, seed):
    from paper_2602_12029_b200 import _lib
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, KVCache, SessionSpec, attn_splits)
    cfg = _cfg(n_layers=2, max_pos=40000)
    n_pages = sum((L + 15) // 16 for L in sess_lens) + sum((p + 16) // 16 for p in priv_lens) + 3
    rng = np.random.default_rng(seed)
    perm = rng.permutation(n_pages).tolist()
    kv = KVCache(cfg, n_pages)
    g = torch.Generator(device="cuda").manual_seed(seed)
    kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
    sessions, rows, ri = [], [], 0
    for s, L in enumerate(sess_lens):
        sessions.append(SessionSpec(shared_len=L, pages=[perm.pop() for _ in range((L + 15) // 16)]))
        for m in range(mods_per_sess[s]):
            rows.append(DecodeRow(module=m, session=s, first_token=0,
                                  pages=[perm.pop() for _ in range((priv_lens[ri] + 16) // 16)]))
            ri += 1
    b = DecodeBatch(sessions, rows, max(mods_per_sess))
    pl = [priv_lens[j] for j in b.order]
    b.t_priv_len.copy_(torch.tensor(pl, dtype=torch.int32))
    R = len(rows)
    q = torch.randn(R, cfg.n_heads, cfg.head_dim, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    splits = attn_splits(b.max_sess_pages + b.max_rps * max((p + 16) // 16 for p in priv_lens),
                         b.n_sess * cfg.n_kv_heads, torch.cuda.get_device_properties(0).multi_processor_count)
    lib = _lib.load()
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_decode_attn_workspace(b.c_ref(), cfg.n_kv_heads, splits, ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value // 4 + 1, dtype=torch.float32, device="cuda")
    layer = 1
    _lib.check(lib.psk_decode_attn(b.c_ref(), q.data_ptr(), cfg.n_heads, layer, kv.layout(), splits,
                                   ws.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    grp = cfg.n_heads // cfg.n_kv_heads
    shared = {}
    for j, row in enumerate(b.rows):
        if row.session not in shared:
            sp = sessions[row.session]
            shared[row.session] = _gather(kv, sp.pages, layer, sp.shared_len)
        ks, vs = shared[row.session]
        kp, vp = _gather(kv, row.pages, layer, pl[j] + 1)
        K = torch.cat([ks, kp], 1).float()
        V = torch.cat([vs, vp], 1).float()
        ref = torch.empty(cfg.n_heads, cfg.head_dim, device="cuda")
        for h in range(cfg.n_heads):
            sc = (K[h // grp] @ q[j, h].float()) / np.sqrt(cfg.head_dim)
            ref[h] = torch.softmax(sc, 0) @ V[h // grp]
        _check(out[j], ref, f"K6 row {j} (session {row.session}, module {row.module})")


def test_k6_fanout_32k_x16_modules():
    """Config 4: 32767 shared tokens read by 16 decode modules (tcgen05 fan-out)."""
    _k6_case([32767], [16], [(i * 37) % 256 for i in range(16)], seed=21)


def test_k6_bench_shape_32_sessions_x4():
    """Config 2 at the bench batch: 32 sessions x 4095 shared tokens x 4 modules."""
    rng = np.random.default_rng(5)
    _k6_case([4095] * 32, [4] * 32, rng.integers(0, 256, 128).tolist(), seed=22)



def test_k3_one_thread_per_row_variant():
    """The K3 variant with one softmax thread per query row
    (PSK_PREFILL_SPLIT=1, read once per process: the K3 cases above rerun in
    a child) matches the fp32 reference as the default two-thread kernel does."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, PSK_PREFILL_SPLIT="1")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", __file__, "-k", "k3 and not variant",
                        "-p", "no:cacheprovider"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
