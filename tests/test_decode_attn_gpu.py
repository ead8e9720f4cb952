"""K6 shared-prefix decode attention vs a torch fp32 reference on identical
bf16 inputs (random paged KV and queries). Covers cluster sizes 1..16,
GQA groups 2/4, 1..16 decode rows per session, several sessions, shared
lengths ending mid-page, empty-ish private suffixes.
Tolerance: |out - ref| <= 2e-2 * max|ref| + 2e-3 (bf16 P in the PV MMA,
bf16 output)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _case(nq, nkv, sess_lens, rows_per_sess, priv_lens, splits, seed=0, dirty_ws=False, ramp=False, reps=1,
          ws=None, b2b=False):
    from paper_2602_12029_b200 import _lib
    from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, KVCache, LlamaConfig,
                                             SessionSpec)
    cfg = LlamaConfig(n_layers=3, d_model=nq * 128, n_heads=nq, n_kv_heads=nkv, ffn=256, vocab=64,
                      rope_theta=1e4, max_pos=65536)
    rng = np.random.default_rng(seed)
    n_pages = sum((L + 15) // 16 for L in sess_lens) + sum((p + 16) // 16 for p in priv_lens) + 3
    perm = list(rng.permutation(n_pages))
    kv = KVCache(cfg, n_pages)
    g = torch.Generator(device="cuda").manual_seed(seed)
    kv.data.copy_(torch.randn(kv.data.shape, device="cuda", generator=g).to(torch.bfloat16))
    if ramp:  # K of later pages scaled up: row maxima grow along the stream (lazy O rescale path)
        pv = kv.page_view()
        for i, pg in enumerate(sorted(set(perm))):
            pv[pg, :, 0] *= 1.0 + 3.0 * (i % 7) / 6.0
    sessions, rows = [], []
    ri = 0
    for s, L in enumerate(sess_lens):
        pages = [perm.pop() for _ in range((L + 15) // 16)]
        sessions.append(SessionSpec(shared_len=L, pages=pages))
        for m in range(rows_per_sess[s]):
            pl = priv_lens[ri]
            rows.append(DecodeRow(module=m, session=s, first_token=0,
                                  pages=[perm.pop() for _ in range((pl + 16) // 16)]))
            ri += 1
    n_mod = max(rows_per_sess)
    b = DecodeBatch(sessions, rows, n_mod)
    pl_by_batch = [priv_lens[j] for j in b.order]
    b.t_priv_len.copy_(torch.tensor(pl_by_batch, dtype=torch.int32))
    R = len(rows)
    q = torch.randn(R, nq, 128, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.full_like(q, float("nan"))
    layer = 1
    import ctypes
    lib = _lib.load()
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_decode_attn_workspace(b.c_ref(), nkv, splits, ctypes.byref(wsb)))
    if ws is None or ws.numel() * 4 < wsb.value:
        ws = torch.zeros(wsb.value // 4 + 1, dtype=torch.float32, device="cuda")
    if dirty_ws:  # stale partials / directory from earlier launches must not leak in
        ws[8192:].uniform_(-50.0, 50.0)  # the leading 32 KiB of merge counters stay zero (API contract)
    for i in range(reps):  # repeated launches reuse the workspace (fused-merge counters reset)
        if not b2b or i == 0:  # b2b: launches back to back (PDL-chained, no other kernel between)
            out.fill_(float("nan"))
        _lib.check(lib.psk_decode_attn(b.c_ref(), q.data_ptr(), nq, layer, kv.layout(), splits,
                                       ws.data_ptr(), out.data_ptr(), torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    grp = nq // nkv
    for j, row in enumerate(b.rows):
        sp = sessions[row.session]
        ks, vs = kv.read_positions(sp.pages, layer, sp.shared_len)
        kp, vp = kv.read_positions(row.pages, layer, pl_by_batch[j] + 1)
        K = torch.cat([ks, kp], 1).float()
        V = torch.cat([vs, vp], 1).float()
        Kq = K.repeat_interleave(grp, 0)
        Vq = V.repeat_interleave(grp, 0)
        sc = (q[j].float().unsqueeze(1) @ Kq.transpose(1, 2)).squeeze(1) / np.sqrt(128)
        ref = (torch.softmax(sc, -1).unsqueeze(1) @ Vq).squeeze(1)
        err = (out[j].float() - ref).abs().max().item()
        assert err <= 2e-2 * ref.abs().max().item() + 2e-3, f"row {j}: err {err}"
    return ws


@pytest.mark.parametrize("splits", [1, 3, 8, 37, 64])
def test_one_session_four_modules(splits):
    _case(32, 8, [4095], [4], [0, 3, 17, 255], splits)


def test_sixteen_modules_fanout():
    """64 query rows per KV head -> the tcgen05 path (> 32 rows)."""
    _case(32, 8, [2000], [16], [i * 7 for i in range(16)], 16, seed=1)


@pytest.mark.parametrize("mods,splits", [(5, 1), (8, 7), (12, 30), (16, 64)])
def test_fanout_tcgen05_shapes(mods, splits):
    """20..64 query rows per KV head (mma.sync up to 32, tcgen05 above), ragged private suffixes,
    shared length ending mid-page, several split counts (incl. splits whose
    last 8-page chunk is partial)."""
    _case(32, 8, [1333], [mods], [(i * 37) % 200 for i in range(mods)], splits, seed=mods)


def test_fanout_fused_merge_reuse():
    """The fan-out kernel's in-kernel merge (one wave of split CTAs): three
    launches on one workspace, then other split counts / groups on the same
    workspace with stale partials; the group counters must come back to zero
    after every launch (arrival counts; the generations advance)."""
    ws = _case(32, 8, [2000], [16], [i * 3 for i in range(16)], 18, seed=5, reps=3)
    ws = _case(32, 8, [900], [16], [i for i in range(16)], 7, seed=6, reps=2, ws=ws, dirty_ws=True)
    ws = _case(32, 8, [300, 77], [16, 9], [i % 20 for i in range(25)], 9, seed=7, reps=2, ws=ws)
    cnt = ws[:8192].view(torch.int32)
    assert (cnt[0::2] & 0xFFFF).sum().item() == 0  # arrivals back to zero
    assert (cnt[0::2] >> 16).sum().item() > 0      # the groups' generations advanced


@pytest.mark.parametrize("lens,splits", [([300], 18), ([40, 70], 9), ([4095], 18)])
def test_fanout_back_to_back(lens, splits):
    """Hundreds of fan-out launches back to back (each PDL-released by the
    previous one, which frees its CTAs' SMs while the rest of its grid is still
    merging): short splits reach the group counters early; they must find them
    re-armed (no lost arrival = no hang, no early pass = exact results)."""
    ws = _case(32, 8, lens, [16] * len(lens), [i * 5 % 37 for i in range(16 * len(lens))], splits, seed=21,
               reps=400, b2b=True)
    cnt = ws[:8192].view(torch.int32)
    assert (cnt[0::2] & 0xFFFF).sum().item() == 0


@pytest.mark.parametrize("lens", [[300] * 20, [37 * i % 900 + 1 for i in range(24)]])
def test_all_heads_back_to_back(lens):
    """The all-heads kernel's in-kernel session merge under hundreds of
    PDL-chained back-to-back launches (see test_fanout_back_to_back)."""
    n = len(lens)
    ws = _case(32, 8, lens, [4] * n, [(3 * i) % 40 for i in range(4 * n)], 1, seed=23, reps=300, b2b=True)
    cnt = ws[:8192].view(torch.int32)
    assert (cnt[0::2] & 0xFFFF).sum().item() == 0


def test_fanout_two_sessions_tcgen05():
    _case(32, 8, [700, 129], [6, 16], [i % 40 for i in range(22)], 9, seed=11)


def test_multi_session_ragged():
    _case(32, 8, [1000, 37, 513], [2, 3, 1], [0, 5, 16, 40, 1, 200], 4, seed=2)


def test_gqa2_tiny_shape():
    _case(2, 1, [99, 300], [2, 2], [0, 1, 15, 31], 2, seed=3)


def test_single_token_shared():
    _case(32, 8, [1], [4], [0, 0, 0, 0], 1, seed=4)


@pytest.mark.parametrize("case", [
    (32, 8, [4095], [4], [0, 3, 17, 255]),
    (32, 8, [4095] * 8, [4] * 8, [255] * 32),                     # the bench shape (8 sessions)
    (32, 8, [1000, 37, 513], [2, 3, 1], [0, 5, 16, 40, 1, 200]),
    (2, 1, [99, 300], [2, 2], [0, 1, 15, 31]),
    (32, 8, [1], [4], [0, 0, 0, 0]),
    (32, 8, [0, 5, 0, 3000], [1, 1, 1, 1], [0, 7, 200, 16]),      # rows without a shared prefix
    (32, 8, [37 * i % 700 for i in range(40)], [1] * 40, [i % 33 for i in range(40)]),  # agent-style
    (32, 8, [12000, 3], [8, 8], [i * 11 for i in range(16)]),     # one long group, one tiny
    (2, 1, [99], [2], [16, 17]),                                   # fewer pages than SMs (empty runs)
])
def test_stream_k_schedule(case):
    """splits = 0: the stream-K partial kernel (runs of equal page counts
    across (session, KV head) groups, segment partials in slot cta + group,
    merge through the group directory) on the shapes above; the fan-out
    (> 32 rows per KV head) sessions fall back to fixed splits."""
    nq, nkv, lens, rps, priv = case
    _case(nq, nkv, lens, rps, priv, 0, seed=len(lens), dirty_ws=True)


@pytest.mark.parametrize("case", [
    (32, 8, [4095] * 20, [4] * 20, [255] * 80),                      # 160 groups: all-heads kernel
    (32, 8, [37 * i % 900 + 1 for i in range(24)], [1, 2, 4] * 8, [(7 * i) % 70 for i in range(56)]),
    (32, 8, [0] * 19 + [300], [1] * 20, [5 * i for i in range(20)]),  # empty shared prefixes
])
def test_all_heads_kernel(case):
    """>= one (session, KV head) group per SM and <= 16 query rows per head:
    the (session, split) all-heads kernel (64 KiB page boxes, warp = head)."""
    nq, nkv, lens, rps, priv = case
    _case(nq, nkv, lens, rps, priv, 1, seed=len(lens))


@pytest.mark.parametrize("mods,splits", [(16, 1), (16, 5), (12, 3), (5, 2)])
def test_growing_scores_rescale(mods, splits):
    """Scores whose maxima grow along the page stream: the fan-out kernel's
    lazy O rescale (and the mma.sync online softmax) under real growth."""
    _case(32, 8, [3000], [mods], [(i * 13) % 100 for i in range(mods)], splits, seed=40 + mods, ramp=True)


@pytest.mark.parametrize("hsplit", ["7", "13"])
def test_all_heads_kernel_forced_splits(hsplit):
    """The all-heads kernel with more (session, split) CTAs than one wave
    (PSK_ATTN_HSPLIT, read once per process: runs the all-heads cases in a
    child) still matches the reference."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, PSK_ATTN_HSPLIT=hsplit)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", __file__, "-k", "test_all_heads_kernel and not forced",
                        "-p", "no:cacheprovider"], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
