"""Drive each hot kernel a few times at the bench shapes, for ncu.

    ncu --set full -k regex:<kernel> -c 2 python tools/profile_kernels.py <which> [rows/module]
which: gemv | gemv_tc | qkv_rope | attn4k | attn4k_s8 | attn4k_s32 | attn32k | gemm | prefill_attn | kvcopy | all
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import ctypes as C  # noqa: E402

import torch  # noqa: E402

from paper_2602_12029_b200 import _lib  # noqa: E402
from paper_2602_12029_b200.model import (DecodeBatch, DecodeRow, KVCache, LlamaConfig,  # noqa: E402
                                         ModuleWeights, PrefillRunner, SessionSpec)

which = sys.argv[1] if len(sys.argv) > 1 else "all"
lib = _lib.load()
s = torch.cuda.current_stream().cuda_stream
cfg = LlamaConfig.llama8b(n_layers=2, max_pos=32768 + 512)


def attn(shared, modules, reps=4, sessions=1):
    n_sh = (shared + 15) // 16
    kv = KVCache(cfg, sessions * (n_sh + modules))
    _lib.check(lib.psk_init_normal_bf16(kv.data.data_ptr(), kv.data.numel(), 7, 1.0, s))
    rows, sess = [], []
    for si in range(sessions):
        base = si * (n_sh + modules)
        sess.append(SessionSpec(shared_len=shared, pages=list(range(base, base + n_sh))))
        rows += [DecodeRow(module=m, session=si, first_token=0, pages=[base + n_sh + m])
                 for m in range(modules)]
    b = DecodeBatch(sess, rows, modules)
    q = torch.randn(sessions * modules, 32, 128, device="cuda").to(torch.bfloat16)
    out = torch.empty_like(q)
    from paper_2602_12029_b200.model import attn_splits
    import os
    ns = attn_splits(n_sh + modules, 8 * sessions, torch.cuda.get_device_properties(0).multi_processor_count)
    if os.environ.get("PSK_SPLITS") is not None:  # 0 = stream-K
        ns = int(os.environ["PSK_SPLITS"])
    wsb = C.c_int64()
    _lib.check(lib.psk_decode_attn_workspace(b.c_ref(), 8, ns, C.byref(wsb)))
    ws = torch.zeros(wsb.value // 4 + 1, dtype=torch.float32, device="cuda")
    for i in range(reps):
        _lib.check(lib.psk_decode_attn(b.c_ref(), q.data_ptr(), 32, i % 2, kv.layout(), ns,
                                       ws.data_ptr(), out.data_ptr(), s))
    torch.cuda.synchronize()


if which in ("attn4k", "all"):
    attn(4095, 4)
if which in ("attn4k_s8", "all"):
    attn(4095, 4, sessions=8)
if which == "attn4k_s32":  # the bench batch: 32 sessions x 4 modules
    attn(4095, 4, sessions=32)
if which in ("attn32k", "all"):
    attn(32767, 16)
if which == "gemv_tc":
    import ctypes
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 32  # rows per module
    mods = [ModuleWeights(cfg, 10 + i) for i in range(4)]
    x = torch.randn(4 * M, cfg.d_model, device="cuda").to(torch.bfloat16)
    act = torch.empty(4 * M, cfg.ffn, dtype=torch.bfloat16, device="cuda")
    hp = (ctypes.c_void_p * 4)(*[m.wgu[0].data_ptr() for m in mods])
    mrs = torch.tensor([i * M for i in range(5)], dtype=torch.int32, device="cuda")
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_gemv_tc_workspace(ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value, dtype=torch.uint8, device="cuda")
    for _ in range(4):
        _lib.check(lib.psk_gemv_tc(x.data_ptr(), 4 * M, cfg.d_model, hp, mrs.data_ptr(), 4, M,
                                   2 * cfg.ffn, 3, act.data_ptr(), ws.data_ptr(), s))
    torch.cuda.synchronize()
if which == "qkv_rope":  # decode QKV GEMV with RoPE + KV append fused (K5-TC epilogue)
    import ctypes
    from paper_2602_12029_b200.model import DecodeBatch as DB, rope_table
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 32  # rows per module
    mods = [ModuleWeights(cfg, 10 + i) for i in range(4)]
    n_sess = M
    kv = KVCache(cfg, n_sess * 4 + 4 * M * 2)
    sess = [SessionSpec(shared_len=40, pages=[4 * i, 4 * i + 1, 4 * i + 2]) for i in range(n_sess)]
    rows = [DecodeRow(module=m, session=i, first_token=0, pages=[4 * n_sess + 2 * (i * 4 + m)])
            for i in range(n_sess) for m in range(4)]
    b = DB(sess, rows, 4)
    x = torch.randn(4 * M, cfg.d_model, device="cuda").to(torch.bfloat16)
    q_rot = torch.empty(4 * M, cfg.n_heads, cfg.head_dim, dtype=torch.bfloat16, device="cuda")
    rope = torch.from_numpy(rope_table(cfg)).cuda()
    hp = (ctypes.c_void_p * 4)(*[m.wqkv[0].data_ptr() for m in mods])
    wsb = ctypes.c_int64()
    _lib.check(lib.psk_gemv_tc_workspace(ctypes.byref(wsb)))
    ws = torch.zeros(wsb.value, dtype=torch.uint8, device="cuda")
    for _ in range(4):
        _lib.check(lib.psk_gemv_tc_qkv_rope(x.data_ptr(), cfg.d_model, hp, b.c_ref(), b.max_rpm, cfg.n_heads,
                                            rope.data_ptr(), 0, kv.layout(), q_rot.data_ptr(), ws.data_ptr(), s))
    torch.cuda.synchronize()
if which == "kvcopy":  # K8: a 4k context's 257 pages (2 MiB each), same-device page copy
    kv = KVCache(LlamaConfig.llama8b(), 2 * 257 + 2)  # all 32 layers: 2 MiB pages
    src = torch.arange(257, dtype=torch.int32, device="cuda")
    dst = torch.arange(257, 514, dtype=torch.int32, device="cuda")
    for _ in range(4):
        _lib.check(lib.psk_kv_copy_pages(kv.data.data_ptr(), kv.data.data_ptr(), src.data_ptr(), dst.data_ptr(), 257,
                                         kv.data[0].numel() * 2, s))
    torch.cuda.synchronize()
if which in ("gemv", "all"):
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # rows per module
    mods = [ModuleWeights(cfg, 10 + i) for i in range(4)]
    x = torch.randn(4 * M, cfg.d_model, device="cuda").to(torch.bfloat16)
    act = torch.empty(4 * M, cfg.ffn, dtype=torch.bfloat16, device="cuda")
    p = torch.tensor([m.wgu[0].data_ptr() for m in mods], dtype=torch.int64, device="cuda")
    mrs = torch.tensor([i * M for i in range(5)], dtype=torch.int32, device="cuda")
    for _ in range(4):
        _lib.check(lib.psk_gemv(x.data_ptr(), 4 * M, cfg.d_model, p.data_ptr(), mrs.data_ptr(), 4, M,
                                2 * cfg.ffn, 3, act.data_ptr(), s))
    torch.cuda.synchronize()
if which in ("gemm", "prefill_attn", "all"):
    base = ModuleWeights(cfg, 3, with_head=False)
    kv = KVCache(cfg, 300)
    pre = PrefillRunner(cfg, base, kv, max_tokens=4096)
    toks = torch.randint(0, cfg.vocab, (4096,), device="cuda")
    pt = torch.arange(256, dtype=torch.int32, device="cuda")
    for _ in range(2):
        pre.run(toks, 0, pt)
    torch.cuda.synchronize()
print("done", which)
