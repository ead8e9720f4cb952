"""Prefill / decode module factorisation on B200 (host side).

Mirrors the reference's module split (frontend/src/model.ts): a frozen base
("prefill module") builds the prompt KV cache once (buildBaseCache,
model.ts:340-352) and task-specific decode modules with the same architecture
but their own weights (train.ts:234, base.clone()) generate from it
(generate with an injected strict-prefix cache, model.ts:363-412). The
architecture is Llama-style (RMSNorm, RoPE rotate-half, GQA, SwiGLU) at the
shapes BASELINE.json names; weights are random-init and generated on the GPU.

All tensor work is done by libpsk.so kernels; torch only owns device memory
and streams.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib

PAGE_TOKENS = 16  # == kvstore block_size
HEAD_DIM = 128


@dataclass(frozen=True)
class LlamaConfig:
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    ffn: int
    vocab: int
    rope_theta: float
    norm_eps: float = 1e-5
    max_pos: int = 8192
    head_dim: int = HEAD_DIM

    @property
    def qkv_dim(self) -> int:
        return (self.n_heads + 2 * self.n_kv_heads) * self.head_dim

    @property
    def page_elems(self) -> int:
        return self.n_layers * 2 * self.n_kv_heads * PAGE_TOKENS * self.head_dim

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * self.n_layers * self.n_kv_heads * self.head_dim * 2

    def param_count(self, with_head: bool = True) -> int:
        d, L = self.d_model, self.n_layers
        per_layer = 2 * d + self.qkv_dim * d + d * self.n_heads * self.head_dim + 3 * self.ffn * d
        return self.vocab * d * (2 if with_head else 1) + L * per_layer + d

    @staticmethod
    def tiny(max_pos: int = 2048) -> "LlamaConfig":
        """BASELINE config 1: 2 layers, d=256 (2 q heads x 128, 1 kv head)."""
        return LlamaConfig(n_layers=2, d_model=256, n_heads=2, n_kv_heads=1, ffn=768, vocab=4096,
                           rope_theta=1e4, max_pos=max_pos)

    @staticmethod
    def llama8b(n_layers: int = 32, max_pos: int = 8192) -> "LlamaConfig":
        """Llama-3.1-8B shape (BASELINE configs 2-5); n_layers < 32 gives the
        full-width truncations used by parity tests."""
        return LlamaConfig(n_layers=n_layers, d_model=4096, n_heads=32, n_kv_heads=8, ffn=14336,
                           vocab=128256, rope_theta=5e5, max_pos=max_pos)


def rope_table(cfg: LlamaConfig) -> np.ndarray:
    """[max_pos][head_dim/2][cos, sin] fp32, computed in float64 (rotate-half
    convention: dims i and i+64 form a pair)."""
    half = cfg.head_dim // 2
    inv = 1.0 / (cfg.rope_theta ** (np.arange(half, dtype=np.float64) * 2.0 / cfg.head_dim))
    ang = np.arange(cfg.max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


def _stream(stream=None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr()


def _mix(*parts: int) -> int:
    x = 0x243F6A8885A308D3
    for p in parts:
        x = (x ^ (p & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        x = (x + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        x = z ^ (z >> 31)
    return x


class ModuleWeights:
    """One module's bf16 weights in the kernels' fused layouts:
    wqkv [q|k|v rows][d]; wgu rows interleaved in 8-row groups
    [gate 8 | up 8], so every 16-row MMA tile of the gate/up GEMV (and
    every 32-column slice of the prefill GEMM) holds matching gate and up
    rows and the epilogue fuses SiLU*mul."""

    def __init__(self, cfg: LlamaConfig, seed: int, device: int = 0, with_head: bool = True,
                 std: float = 0.02):
        self.cfg = cfg
        self.seed = seed
        dev = torch.device("cuda", device)
        bf = torch.bfloat16
        d = cfg.d_model
        self.embed = torch.empty(cfg.vocab, d, dtype=bf, device=dev)
        self.attn_norm, self.wqkv, self.wo, self.mlp_norm, self.wgu, self.wdown = [], [], [], [], [], []
        for _ in range(cfg.n_layers):
            self.attn_norm.append(torch.empty(d, dtype=bf, device=dev))
            self.wqkv.append(torch.empty(cfg.qkv_dim, d, dtype=bf, device=dev))
            self.wo.append(torch.empty(d, cfg.n_heads * cfg.head_dim, dtype=bf, device=dev))
            self.mlp_norm.append(torch.empty(d, dtype=bf, device=dev))
            self.wgu.append(torch.empty(2 * cfg.ffn, d, dtype=bf, device=dev))
            self.wdown.append(torch.empty(d, cfg.ffn, dtype=bf, device=dev))
        self.final_norm = torch.empty(d, dtype=bf, device=dev)
        self.head = torch.empty(cfg.vocab, d, dtype=bf, device=dev) if with_head else None
        s = _stream()
        lib = _lib.load()
        for i, (t, kind) in enumerate(self._tensors()):
            tseed = _mix(seed, i)
            if kind == "norm":
                # gammas ~ 1 + N(0, 0.1): exercises the per-module gamma path
                _lib.check(lib.psk_init_normal_bf16(_ptr(t), t.numel(), tseed, 0.1, s))
                t.add_(1.0)
            else:
                _lib.check(lib.psk_init_normal_bf16(_ptr(t), t.numel(), tseed, std, s))

    def _tensors(self):
        out = [(self.embed, "w")]
        for l in range(self.cfg.n_layers):
            out += [(self.attn_norm[l], "norm"), (self.wqkv[l], "w"), (self.wo[l], "w"),
                    (self.mlp_norm[l], "norm"), (self.wgu[l], "w"), (self.wdown[l], "w")]
        out.append((self.final_norm, "norm"))
        if self.head is not None:
            out.append((self.head, "w"))
        return out

    def nbytes(self) -> int:
        return sum(t.numel() * 2 for t, _ in self._tensors())

    def layer_bytes(self) -> int:
        """Weight bytes one decode step streams per module (all layers + head)."""
        c = self.cfg
        per_layer = (c.qkv_dim * c.d_model + c.d_model * c.n_heads * c.head_dim +
                     3 * c.ffn * c.d_model + 2 * c.d_model) * 2
        return c.n_layers * per_layer + (c.vocab * c.d_model * 2 if self.head is not None else 0)

    def layer_reference(self, l: int) -> dict:
        """fp32 CPU copy of layer l in the standard (un-fused) layout, for the
        oracle (test infrastructure; full-size parity streams layers one at
        a time so host memory stays near one layer)."""
        c = self.cfg
        f = lambda t: t.cpu().float()  # noqa: E731
        qd, kd = c.n_heads * c.head_dim, c.n_kv_heads * c.head_dim
        qkv = f(self.wqkv[l])
        gu = f(self.wgu[l]).view(-1, 2, 8, c.d_model)
        return {"attn_norm": f(self.attn_norm[l]), "wq": qkv[:qd], "wk": qkv[qd:qd + kd],
                "wv": qkv[qd + kd:], "wo": f(self.wo[l]), "mlp_norm": f(self.mlp_norm[l]),
                "w_gate": gu[:, 0].reshape(c.ffn, c.d_model),
                "w_up": gu[:, 1].reshape(c.ffn, c.d_model),
                "w_down": f(self.wdown[l])}

    def reference_layout(self) -> dict:
        """fp32 CPU copies in the standard (un-fused) layout, for the oracle."""
        f = lambda t: t.cpu().float()  # noqa: E731
        out = {"embed": f(self.embed), "final_norm": f(self.final_norm),
               "layers": [self.layer_reference(l) for l in range(self.cfg.n_layers)]}
        if self.head is not None:
            out["head"] = f(self.head)
        return out


class KVCache:
    """Paged KV memory: bf16 [n_pages][layer][K|V][kv_head][16][128]."""

    def __init__(self, cfg: LlamaConfig, n_pages: int, device: int = 0):
        self.cfg = cfg
        self.n_pages = n_pages
        self.data = torch.zeros(n_pages, cfg.page_elems, dtype=torch.bfloat16,
                                device=torch.device("cuda", device))

    def layout(self) -> "KVLayout":
        c = self.cfg
        return KVLayout(self.data.data_ptr(), c.page_elems, c.n_layers, c.n_kv_heads, c.head_dim,
                        PAGE_TOKENS, self.n_pages)

    def page_view(self) -> torch.Tensor:
        c = self.cfg
        return self.data.view(self.n_pages, c.n_layers, 2, c.n_kv_heads, PAGE_TOKENS, c.head_dim)

    def write_positions(self, pages: list[int], layer: int, k: torch.Tensor, v: torch.Tensor,
                        start: int = 0) -> None:
        """Test / transfer plumbing: write K,V [n_kv, T, hd] for positions
        start..start+T-1 of a page table (not on any hot path)."""
        pv = self.page_view()
        T = k.shape[1]
        for t in range(T):
            p = start + t
            pg = pages[p // PAGE_TOKENS]
            pv[pg, layer, 0, :, p % PAGE_TOKENS] = k[:, t].to(pv.dtype)
            pv[pg, layer, 1, :, p % PAGE_TOKENS] = v[:, t].to(pv.dtype)

    def read_positions(self, pages: list[int], layer: int, n: int, start: int = 0):
        pv = self.page_view()
        ks, vs = [], []
        for t in range(n):
            p = start + t
            pg = pages[p // PAGE_TOKENS]
            ks.append(pv[pg, layer, 0, :, p % PAGE_TOKENS])
            vs.append(pv[pg, layer, 1, :, p % PAGE_TOKENS])
        if n == 0:
            e = pv.new_empty(pv.shape[3], 0, pv.shape[5])
            return e, e.clone()
        return torch.stack(ks, 1), torch.stack(vs, 1)


KVLayout = _lib.KVLayout
DecodeBatchC = _lib.DecodeBatchC


@dataclass
class DecodeRow:
    module: int          # index into the runner's module list
    session: int         # index into the batch's sessions
    first_token: int     # last prompt token (the module processes it itself)
    pages: list[int]     # private KV pages (capacity for max_new tokens)


@dataclass
class SessionSpec:
    shared_len: int      # base-prefill positions the rows attend to: n - 1
    pages: list[int]     # shared KV page table (covers shared_len positions)


class DecodeBatch:
    """Device arrays describing a set of decode rows (psk_decode_batch)."""

    def __init__(self, sessions: list[SessionSpec], rows: list[DecodeRow], n_modules: int,
                 device: int = 0):
        dev = torch.device("cuda", device)
        for i, sp in enumerate(sessions):  # the kernels read ceil(shared_len / 16) page ids of each session
            if sp.shared_len < 0 or (sp.shared_len + PAGE_TOKENS - 1) // PAGE_TOKENS > len(sp.pages):
                raise ValueError(f"session {i}: {len(sp.pages)} pages cannot hold shared_len {sp.shared_len}")
        order = sorted(range(len(rows)), key=lambda i: (rows[i].module, i))
        self.rows = [rows[i] for i in order]
        self.order = order  # batch row j is caller row order[j]
        self.mod_ids = sorted({r.module for r in self.rows})
        mod_index = {m: i for i, m in enumerate(self.mod_ids)}
        R, S = len(self.rows), len(sessions)
        mrs = [0] * (len(self.mod_ids) + 1)
        for r in self.rows:
            mrs[mod_index[r.module] + 1] += 1
        for i in range(len(self.mod_ids)):
            mrs[i + 1] += mrs[i]
        sess_rows: list[list[int]] = [[] for _ in range(S)]
        row_in_sess = []
        for j, r in enumerate(self.rows):
            row_in_sess.append(len(sess_rows[r.session]))
            sess_rows[r.session].append(j)
        self.max_rps = max(1, max(len(x) for x in sess_rows))
        self.max_rpm = max(mrs[i + 1] - mrs[i] for i in range(len(self.mod_ids)))  # rows per module
        msp = max(1, max(len(s.pages) for s in sessions))
        mrp = max(1, max(len(r.pages) for r in self.rows))
        i32 = lambda x: torch.tensor(x, dtype=torch.int32, device=dev)  # noqa: E731
        self.t_row_mod = i32([mod_index[r.module] for r in self.rows])
        self.t_row_sess = i32([r.session for r in self.rows])
        self.t_row_in_sess = i32(row_in_sess)
        self.t_mrs = i32(mrs)
        self.t_sess_rows = i32([x + [0] * (self.max_rps - len(x)) for x in sess_rows])
        self.t_sess_nrows = i32([len(x) for x in sess_rows])
        self.t_sess_len = i32([s.shared_len for s in sessions])
        self.t_sess_pages = i32([s.pages + [0] * (msp - len(s.pages)) for s in sessions])
        self.t_row_pages = i32([r.pages + [0] * (mrp - len(r.pages)) for r in self.rows])
        self.t_priv_len = i32([0] * R)
        self.t_tokens = i32([r.first_token for r in self.rows])
        self.n_rows, self.n_sess, self.n_mod = R, S, len(self.mod_ids)
        self.c = DecodeBatchC(
            R, S, len(self.mod_ids), self.max_rps,
            _ptr(self.t_row_mod), _ptr(self.t_row_sess), _ptr(self.t_row_in_sess), _ptr(self.t_mrs),
            _ptr(self.t_sess_rows), _ptr(self.t_sess_nrows), _ptr(self.t_sess_len),
            _ptr(self.t_sess_pages), msp, _ptr(self.t_row_pages), mrp,
            _ptr(self.t_priv_len), _ptr(self.t_tokens))

        self.max_sess_pages = msp
        self._first = [r.first_token for r in self.rows]

    def c_ref(self):
        return C.byref(self.c)

    def reset(self) -> None:
        self.t_priv_len.zero_()
        self.t_tokens.copy_(torch.tensor(self._first, dtype=torch.int32))

    def update_row(self, row: int, shared_len: int, pages: list[int], first_token: int) -> None:
        """Re-point one row (that is also its own session) at a new request
        in place, ordered on the current stream: continuous batching."""
        msp = self.max_sess_pages
        if len(pages) > msp:
            raise ValueError("row page table exceeds the batch's capacity")
        s = self.rows[row].session
        self.t_sess_len[s] = shared_len
        # pinned staging + async copy: no stream sync (the caching host
        # allocator keeps the pinned block alive until the copy has run)
        host = torch.tensor(pages + [pages[-1]] * (msp - len(pages)), dtype=torch.int32).pin_memory()
        self.t_sess_pages[s].copy_(host, non_blocking=True)
        self.t_priv_len[row] = 0
        self.t_tokens[row] = first_token
        self._first[row] = first_token

    def update_sessions(self, shared_lens: list[int], pages: list[list[int]],
                        first_tokens: list[int]) -> None:
        """Point the batch at new sessions in place (same device addresses, so
        a captured decode graph stays valid). first_tokens: per session (the
        session's last prompt token, which every module processes itself)."""
        msp = self.max_sess_pages
        if any(len(p) > msp for p in pages):
            raise ValueError("session page table exceeds the batch's capacity")
        self.t_sess_len.copy_(torch.tensor(shared_lens, dtype=torch.int32))
        self.t_sess_pages.copy_(torch.tensor([p + [0] * (msp - len(p)) for p in pages], dtype=torch.int32))
        self._first = [first_tokens[r.session] for r in self.rows]
        self.reset()


def batch_plan(cfg: LlamaConfig, seqs) -> tuple[np.ndarray, int]:
    """Device plan of a batched partial prefill (run_batch / K3 batch form).
    seqs: list of (new tokens T_i, pos0_i, page table covering [0, pos0_i+T_i)).
    Returns (int32 array [items x 8 | row positions | row KV slots | pages],
    number of work items). A work item is one (sequence, 256/grp-row q-block):
    (row offset, T_i, pos0_i, page offset, q-block, 0, 0, 0), sorted heaviest
    (longest key range) first."""
    grp = cfg.n_heads // cfg.n_kv_heads
    qb = 256 // grp
    row_pos, row_slot, pages, items = [], [], [], []
    off = 0
    for n, pos0, pt in seqs:
        if pos0 + n > cfg.max_pos:
            raise ValueError(f"sequence length {pos0 + n} exceeds max_pos {cfg.max_pos}")
        ptn = (pt.cpu().numpy() if torch.is_tensor(pt) else np.asarray(pt)).astype(np.int64)
        pos = np.arange(pos0, pos0 + n, dtype=np.int64)
        row_pos.append(pos)
        row_slot.append(ptn[pos // PAGE_TOKENS] * PAGE_TOKENS + pos % PAGE_TOKENS)
        for k in range((n + qb - 1) // qb):
            kv_end = pos0 + min((k + 1) * qb, n)
            items.append((kv_end, [off, n, pos0, len(pages), k, 0, 0, 0]))
        pages.extend(ptn.tolist())
        off += n
    items.sort(key=lambda x: -x[0])  # heaviest (longest key range) first
    # items first: the kernel reads them as int4 (16-byte aligned)
    plan = np.concatenate([np.asarray([it for _, it in items], dtype=np.int64).reshape(-1),
                           np.concatenate(row_pos), np.concatenate(row_slot),
                           np.asarray(pages, dtype=np.int64)]).astype(np.int32)
    return plan, len(items)


PER_SEQ_ATTN_MIN_TOKENS = 1024  # batched prefill: per-sequence K3 when every sequence has this many new tokens
GEMV_MMA_MAX_ROWS = 8  # rows per module up to which the mma.sync GEMV (K5) beats K5-TC


def attn_splits(max_pages: int, n_groups: int, sms: int = 148) -> int:
    """Split-KV factor for K6: one CTA per SM over the (session, KV head)
    groups, at least ~4 pages per split, at most 512 splits."""
    return max(1, min(sms // max(1, n_groups), max(1, max_pages // 4), 512))


class DecodeRunner:
    """Runs greedy decode steps for a DecodeBatch of heterogeneous modules.

    One step = embed -> L x [RMSNorm, grouped QKV GEMV, RoPE + KV append,
    shared-prefix attention (K6), O GEMV (+residual), RMSNorm, gate/up GEMV
    (+SiLU*mul), down GEMV (+residual)] -> RMSNorm -> LM head GEMV -> argmax.
    The step is captured once into a CUDA graph and replayed.
    """

    def __init__(self, cfg: LlamaConfig, modules: list[ModuleWeights], kv: KVCache,
                 batch: DecodeBatch, max_new: int, splits: int | None = None, device: int = 0):
        self.cfg, self.kv, self.b, self.max_new = cfg, kv, batch, max_new
        self.lib = _lib.load()
        dev = torch.device("cuda", device)
        mods = [modules[m] for m in batch.mod_ids]
        ptrs = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)  # noqa: E731
        L = cfg.n_layers
        self.p_embed = ptrs([m.embed for m in mods])
        self.p_attn_norm = [ptrs([m.attn_norm[l] for m in mods]) for l in range(L)]
        self.p_wqkv = [ptrs([m.wqkv[l] for m in mods]) for l in range(L)]
        self.p_wo = [ptrs([m.wo[l] for m in mods]) for l in range(L)]
        self.p_mlp_norm = [ptrs([m.mlp_norm[l] for m in mods]) for l in range(L)]
        self.p_wgu = [ptrs([m.wgu[l] for m in mods]) for l in range(L)]
        self.p_wdown = [ptrs([m.wdown[l] for m in mods]) for l in range(L)]
        self.p_final_norm = ptrs([m.final_norm for m in mods])
        self.p_head = ptrs([m.head for m in mods])
        # > 8 rows per module: the tcgen05 GEMV (K5-TC) takes host pointer arrays
        self.use_tc_gemv = batch.max_rpm > GEMV_MMA_MAX_ROWS
        hptrs = lambda ts: (C.c_void_p * len(ts))(*[t.data_ptr() for t in ts])  # noqa: E731
        self.h_wqkv = [hptrs([m.wqkv[l] for m in mods]) for l in range(L)]
        self.h_wo = [hptrs([m.wo[l] for m in mods]) for l in range(L)]
        self.h_wgu = [hptrs([m.wgu[l] for m in mods]) for l in range(L)]
        self.h_wdown = [hptrs([m.wdown[l] for m in mods]) for l in range(L)]
        self.h_head = hptrs([m.head for m in mods])
        gwb = C.c_int64()
        _lib.check(self.lib.psk_gemv_tc_workspace(C.byref(gwb)))
        self.gemv_ws = torch.zeros(gwb.value, dtype=torch.uint8, device=dev)  # flags start (and end) at 0
        self.weight_bytes_per_step = sum(m.layer_bytes() for m in mods)
        R, d = batch.n_rows, cfg.d_model
        f32, bf = torch.float32, torch.bfloat16
        self.h = torch.empty(R, d, dtype=f32, device=dev)
        self.xn = torch.empty(R, d, dtype=bf, device=dev)
        self.qkv = torch.empty(R, cfg.qkv_dim, dtype=f32, device=dev)
        self.q_rot = torch.empty(R, cfg.n_heads, cfg.head_dim, dtype=bf, device=dev)
        self.attn = torch.empty(R, cfg.n_heads * cfg.head_dim, dtype=bf, device=dev)
        self.act = torch.empty(R, cfg.ffn, dtype=bf, device=dev)
        self.logits = torch.empty(R, cfg.vocab, dtype=f32, device=dev)
        self.out_tokens = torch.full((R, max_new), -1, dtype=torch.int32, device=dev)
        self.rope = torch.from_numpy(rope_table(cfg)).to(dev)
        sms = _lib.sm_budget()  # the SMs this runner's kernels are sized for
        # fixed splits (one CTA per SM over the groups). splits=0 selects the
        # stream-K schedule of K6, which is correct but measured slower: runs
        # that cut across (session, head) groups lose the DRAM locality of 8
        # heads' CTAs reading the same pages together
        self.splits = splits if splits is not None else attn_splits(
            batch.max_sess_pages + batch.max_rps * ((max_new + 15) // 16),
            batch.n_sess * cfg.n_kv_heads, sms)
        wsb = C.c_int64()
        _lib.check(self.lib.psk_decode_attn_workspace(batch.c_ref(), cfg.n_kv_heads, self.splits,
                                                      C.byref(wsb)))
        self.ws = torch.zeros(wsb.value // 4 + 1, dtype=f32, device=dev)  # split counters start at 0
        self.graph: torch.cuda.CUDAGraph | None = None
        # K5-TC: RoPE + KV append fused into the QKV GEMV's epilogue (one
        # launch instead of two per layer) with PSK_FUSED_QKV=1. Bit-identical
        # but not faster: at 32 rows/module the step is 13.36-13.38 ms fused
        # vs 13.35-13.37 ms apart (the epilogue's head-pair exchange and row
        # table sit on the stream-K owners' critical path), so it is off
        self.fused_qkv = self.use_tc_gemv and os.environ.get("PSK_FUSED_QKV", "0") == "1"
        # K5-TC: the o-proj / down-proj residual GEMVs also write the next
        # RMSNorm's output (psk_gemv_tc_resid_norm) with PSK_FUSED_NORM=1.
        # Correct but slower: the in-kernel grid barrier over a module's
        # units holds every CTA until the slowest, so the next GEMV can no
        # longer stream its weights under this one's tail (13.68-13.69 vs
        # 13.32-13.36 ms per step at 32 rows/module); off by default
        self.fused_norm = self.use_tc_gemv and os.environ.get("PSK_FUSED_NORM", "0") == "1"
        # K6 launches 1 kernel when the fan-out kernel merges its splits
        # itself, else 2 (partial + merge)
        n_attn = C.c_int32()
        _lib.check(self.lib.psk_decode_attn_kernels(batch.c_ref(), cfg.n_heads, cfg.n_kv_heads, self.splits,
                                                    C.byref(n_attn)))
        norm_fused = self.fused_norm and batch.n_mod * (cfg.d_model // 128) <= sms and batch.max_rpm <= 64
        # embed, L x [norm, qkv, rope, attention, o, norm, gate/up, down], final norm, head, argmax; the
        # fused norms drop 2 launches per layer (layer 0's norm stays, the final norm rides the last down GEMV)
        self.launches_per_step = 1 + L * (7 + n_attn.value - self.fused_qkv - 2 * norm_fused) + 3

    def _gemv(self, x, K: int, p_dev, p_host, N: int, epi: int, out, s: int) -> None:
        """K5 (mma.sync, <= 8 rows per module) or K5-TC (tcgen05, 9..64)."""
        b = self.b
        if self.use_tc_gemv:
            _lib.check(self.lib.psk_gemv_tc(_ptr(x), b.n_rows, K, p_host, _ptr(b.t_mrs), b.n_mod, b.max_rpm, N,
                                            epi, _ptr(out), _ptr(self.gemv_ws), s))
        else:
            _lib.check(self.lib.psk_gemv(_ptr(x), b.n_rows, K, _ptr(p_dev), _ptr(b.t_mrs), b.n_mod, b.max_rpm, N,
                                         epi, _ptr(out), s))

    def _gemv_norm(self, x, K: int, p_host, gamma, s: int) -> None:
        """K5-TC residual GEMV (h += W x) + the next RMSNorm (xn) in one call."""
        b, cfg = self.b, self.cfg
        _lib.check(self.lib.psk_gemv_tc_resid_norm(_ptr(x), b.n_rows, K, p_host, _ptr(b.t_mrs), b.n_mod, b.max_rpm,
                                                   cfg.d_model, _ptr(self.h), _ptr(gamma), _ptr(b.t_row_mod),
                                                   C.c_float(cfg.norm_eps), _ptr(self.xn), _ptr(self.gemv_ws), s))

    # -- one step, eager ----------------------------------------------------
    def _step(self, s: int) -> None:
        lib, cfg, b = self.lib, self.cfg, self.b
        bc = C.byref(b.c)
        R, d = b.n_rows, cfg.d_model
        kvl = self.kv.layout()
        chk = _lib.check
        gemv = self._gemv
        chk(lib.psk_embed_rows(bc, _ptr(self.p_embed), d, _ptr(self.h), s))
        for l in range(cfg.n_layers):
            if l == 0 or not self.fused_norm:  # (fused: the previous down GEMV wrote this norm)
                chk(lib.psk_rmsnorm_rows(_ptr(self.h), R, d, _ptr(self.p_attn_norm[l]), _ptr(b.t_row_mod),
                                         C.c_float(cfg.norm_eps), _ptr(self.xn), s))
            if self.fused_qkv:
                chk(lib.psk_gemv_tc_qkv_rope(_ptr(self.xn), d, self.h_wqkv[l], bc, b.max_rpm, cfg.n_heads,
                                             _ptr(self.rope), l, kvl, _ptr(self.q_rot), _ptr(self.gemv_ws), s))
            else:
                gemv(self.xn, d, self.p_wqkv[l], self.h_wqkv[l], cfg.qkv_dim, 1, self.qkv, s)
                chk(lib.psk_rope_append(bc, _ptr(self.qkv), cfg.n_heads, _ptr(self.rope), l, kvl,
                                        _ptr(self.q_rot), s))
            chk(lib.psk_decode_attn(bc, _ptr(self.q_rot), cfg.n_heads, l, kvl, self.splits,
                                    _ptr(self.ws), _ptr(self.attn), s))
            if self.fused_norm:  # residual GEMV + the MLP norm in one launch
                self._gemv_norm(self.attn, cfg.n_heads * cfg.head_dim, self.h_wo[l], self.p_mlp_norm[l], s)
            else:
                gemv(self.attn, cfg.n_heads * cfg.head_dim, self.p_wo[l], self.h_wo[l], d, 2, self.h, s)
                chk(lib.psk_rmsnorm_rows(_ptr(self.h), R, d, _ptr(self.p_mlp_norm[l]), _ptr(b.t_row_mod),
                                         C.c_float(cfg.norm_eps), _ptr(self.xn), s))
            gemv(self.xn, d, self.p_wgu[l], self.h_wgu[l], 2 * cfg.ffn, 3, self.act, s)
            nxt = self.p_attn_norm[l + 1] if l + 1 < cfg.n_layers else self.p_final_norm
            if self.fused_norm:  # residual GEMV + the next layer's attention norm (or the final norm)
                self._gemv_norm(self.act, cfg.ffn, self.h_wdown[l], nxt, s)
            else:
                gemv(self.act, cfg.ffn, self.p_wdown[l], self.h_wdown[l], d, 2, self.h, s)
        if not self.fused_norm:
            chk(lib.psk_rmsnorm_rows(_ptr(self.h), R, d, _ptr(self.p_final_norm), _ptr(b.t_row_mod),
                                     C.c_float(cfg.norm_eps), _ptr(self.xn), s))
        gemv(self.xn, d, self.p_head, self.h_head, cfg.vocab, 1, self.logits, s)
        chk(lib.psk_argmax_advance(bc, _ptr(self.logits), cfg.vocab, _ptr(self.out_tokens),
                                   self.max_new, s))

    def capture(self) -> None:
        """Capture one step into a CUDA graph (lengths live on the device)."""
        self.b.reset()
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(st):
            self._step(st.cuda_stream)  # warm-up (sets kernel attributes)
        torch.cuda.current_stream().wait_stream(st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self._step(torch.cuda.current_stream().cuda_stream)
        self.graph = g
        torch.cuda.synchronize()

    def run(self, n_steps: int, use_graph: bool = True) -> torch.Tensor:
        """Reset and generate n_steps tokens per row; returns out_tokens in the
        caller's row order."""
        self.b.reset()
        self.out_tokens.fill_(-1)
        if use_graph and self.graph is None:
            self.capture()
            self.b.reset()
            self.out_tokens.fill_(-1)
        for _ in range(n_steps):
            if use_graph:
                self.graph.replay()
            else:
                self._step(_stream())
        inv = torch.empty_like(self.out_tokens)
        inv[torch.tensor(self.b.order, device=self.out_tokens.device)] = self.out_tokens
        return inv


class PrefillRunner:
    """The frozen prefill module: buildBaseCache (model.ts:340-352) on B200.

    Forwards the new prompt tokens [pos0, pos0+T) through all layers and
    leaves their K/V in the paged cache (fused into the QKV GEMM epilogue).
    No final norm / LM head: the prefill module's own next token is never
    used ((., C_base) = F(X, 0)).
    Per layer: RMSNorm -> QKV GEMM (+RoPE, paged KV write) -> causal paged
    attention -> O GEMM (+residual) -> RMSNorm -> gate/up GEMM (+SiLU*mul)
    -> down GEMM (+residual).
    """

    def __init__(self, cfg: LlamaConfig, weights: ModuleWeights, kv: KVCache, max_tokens: int,
                 device: int = 0):
        self.cfg, self.w, self.kv = cfg, weights, kv
        self.lib = _lib.load()
        dev = torch.device("cuda", device)
        d = cfg.d_model
        self.max_tokens = max_tokens
        f32, bf = torch.float32, torch.bfloat16
        self.h = torch.empty(max_tokens, d, dtype=f32, device=dev)
        self.xn = torch.empty(max_tokens, d, dtype=bf, device=dev)
        self.q = torch.empty(max_tokens, cfg.n_heads, cfg.head_dim, dtype=bf, device=dev)
        self.attn = torch.empty(max_tokens, cfg.n_heads * cfg.head_dim, dtype=bf, device=dev)
        self.act = torch.empty(max_tokens, cfg.ffn, dtype=bf, device=dev)
        self.rope = torch.from_numpy(rope_table(cfg)).to(dev)
        self.gamma_ptrs = [
            (torch.tensor([weights.attn_norm[l].data_ptr()], dtype=torch.int64, device=dev),
             torch.tensor([weights.mlp_norm[l].data_ptr()], dtype=torch.int64, device=dev))
            for l in range(cfg.n_layers)]
        self.launches_per_call = 1 + 7 * cfg.n_layers
        # (the GEMMs' split-K tail, psk_gemm_bind_workspace, is left unbound:
        # measured slower end to end at the 4k prefill shapes)

    def flops(self, T: int, pos0: int = 0) -> float:
        """Algorithmic FLOPs of one call (GEMMs + causal attention)."""
        c = self.cfg
        gemm = 2.0 * T * c.n_layers * (c.qkv_dim * c.d_model + c.d_model * c.n_heads * c.head_dim +
                                       3 * c.ffn * c.d_model)
        # causal: query i (absolute pos0+i) sees pos0+i+1 keys
        keys = T * pos0 + T * (T + 1) / 2.0
        attn = 4.0 * c.n_layers * c.n_heads * c.head_dim * keys
        return gemm + attn

    def run(self, tokens: torch.Tensor, pos0: int, page_table: torch.Tensor, stream: int | None = None,
            kv_only: bool = False) -> None:
        """tokens: int64 device [T] (the same ids the block pool hashes);
        page_table: int32 device covering positions [0, pos0+T).
        kv_only: stop after the last layer's QKV GEMM (its K/V written). A
        prefill that only builds the shared cache (buildBaseCache,
        model.ts:340; the decode modules process the last prompt token
        themselves) never reads the last layer's attention / MLP output, so
        the KV pages are identical and ~1/32 of the forward is skipped."""
        cfg, lib, w = self.cfg, self.lib, self.w
        T = int(tokens.shape[0])
        if T > self.max_tokens:
            raise ValueError(f"prefill of {T} tokens exceeds max_tokens {self.max_tokens}")
        if pos0 + T > cfg.max_pos:
            raise ValueError(f"sequence length {pos0 + T} exceeds max_pos {cfg.max_pos}")
        s = stream if stream is not None else _stream()
        chk = _lib.check
        d = cfg.d_model
        kvl = self.kv.layout()
        pt = _ptr(page_table)
        eps = C.c_float(cfg.norm_eps)
        chk(lib.psk_embed_tokens(_ptr(tokens), T, _ptr(w.embed), d, _ptr(self.h), s))
        for l in range(cfg.n_layers):
            g1, g2 = self.gamma_ptrs[l]
            chk(lib.psk_rmsnorm_rows(_ptr(self.h), T, d, _ptr(g1), None, eps, _ptr(self.xn), s))
            chk(lib.psk_gemm_qkv_rope_kv(_ptr(self.xn), _ptr(w.wqkv[l]), T, d, cfg.n_heads,
                                         _ptr(self.rope), pos0, kvl, l, pt, _ptr(self.q), s))
            if kv_only and l == cfg.n_layers - 1:
                break
            chk(lib.psk_prefill_attn(_ptr(self.q), T, pos0, cfg.n_heads, kvl, l, pt, _ptr(self.attn), s))
            chk(lib.psk_gemm(_ptr(self.attn), _ptr(w.wo[l]), T, d, cfg.n_heads * cfg.head_dim, 2,
                             _ptr(self.h), d, s))
            chk(lib.psk_rmsnorm_rows(_ptr(self.h), T, d, _ptr(g2), None, eps, _ptr(self.xn), s))
            chk(lib.psk_gemm(_ptr(self.xn), _ptr(w.wgu[l]), T, 2 * cfg.ffn, d, 3, _ptr(self.act),
                             cfg.ffn, s))
            chk(lib.psk_gemm(_ptr(self.act), _ptr(w.wdown[l]), T, d, cfg.ffn, 2, _ptr(self.h), d, s))

    def run_batch(self, seqs, stream: int | None = None, kv_only: bool = False) -> None:
        """Batched partial prefill: the new tokens of several
        sequences in ONE forward, so the (weight-bound) small prefills of an
        agent workload share each layer's weight stream. seqs: list of
        (tokens int64 device [T_i], pos0_i, page table covering [0, pos0_i+T_i)
        as a list / int32 tensor). Rows are stacked; the QKV epilogue places
        each row's K/V by its own (position, slot) and K3 runs one CTA per
        (sequence, q-block, KV head)."""
        if len(seqs) == 1:
            toks, pos0, pt = seqs[0]
            if not torch.is_tensor(pt):
                pt = torch.tensor(pt, dtype=torch.int32, device=self.h.device)
            return self.run(toks, pos0, pt, stream, kv_only)
        cfg, lib, w = self.cfg, self.lib, self.w
        Ts = [int(t.shape[0]) for t, _, _ in seqs]
        T = sum(Ts)
        if T > self.max_tokens:
            raise ValueError(f"batched prefill of {T} tokens exceeds max_tokens {self.max_tokens}")
        plan, n_items = batch_plan(cfg, [(n, pos0, pt) for (_, pos0, pt), n in zip(seqs, Ts)])
        dplan = torch.from_numpy(plan).to(self.h.device)
        ni = 8 * n_items
        d_items = dplan[:ni]
        d_pos, d_slot = dplan[ni:ni + T], dplan[ni + T:ni + 2 * T]
        d_pages = dplan[ni + 2 * T:]
        tokens = torch.cat([t for t, _, _ in seqs])
        # >= 1024 new tokens in every sequence: per-sequence K3 launches (the
        # single-sequence kernel's 128-row ping-pong tiles beat the batched
        # kernel's 64-token q-blocks there); GEMMs stay batched
        per_seq = []
        if min(Ts) >= PER_SEQ_ATTN_MIN_TOKENS:
            o_, pg_ = 0, 0
            for (_, pos0, pt), n in zip(seqs, Ts):
                per_seq.append((o_, n, pos0, pg_))
                o_ += n
                pg_ += len(pt)
        qrow = cfg.n_heads * cfg.head_dim * 2  # bytes per token row of q / attn
        self._batch_keep = (dplan, tokens)  # alive until the next call (async kernels)
        s = stream if stream is not None else _stream()
        chk = _lib.check
        d = cfg.d_model
        kvl = self.kv.layout()
        eps = C.c_float(cfg.norm_eps)
        chk(lib.psk_embed_tokens(_ptr(tokens), T, _ptr(w.embed), d, _ptr(self.h), s))
        for l in range(cfg.n_layers):
            g1, g2 = self.gamma_ptrs[l]
            chk(lib.psk_rmsnorm_rows(_ptr(self.h), T, d, _ptr(g1), None, eps, _ptr(self.xn), s))
            chk(lib.psk_gemm_qkv_rope_kv_rows(_ptr(self.xn), _ptr(w.wqkv[l]), T, d, cfg.n_heads,
                                              _ptr(self.rope), _ptr(d_pos), _ptr(d_slot), kvl, l,
                                              _ptr(self.q), s))
            if kv_only and l == cfg.n_layers - 1:
                break
            if per_seq:  # long sequences: the single-sequence ping-pong K3 on each row range
                for (o_, n_, p0_, pg_) in per_seq:
                    chk(lib.psk_prefill_attn(_ptr(self.q) + o_ * qrow, n_, p0_, cfg.n_heads, kvl, l,
                                             _ptr(d_pages) + 4 * pg_, _ptr(self.attn) + o_ * qrow, s))
            else:
                chk(lib.psk_prefill_attn_batch(_ptr(self.q), n_items, _ptr(d_items), cfg.n_heads, kvl, l,
                                               _ptr(d_pages), _ptr(self.attn), s))
            chk(lib.psk_gemm(_ptr(self.attn), _ptr(w.wo[l]), T, d, cfg.n_heads * cfg.head_dim, 2,
                             _ptr(self.h), d, s))
            chk(lib.psk_rmsnorm_rows(_ptr(self.h), T, d, _ptr(g2), None, eps, _ptr(self.xn), s))
            chk(lib.psk_gemm(_ptr(self.xn), _ptr(w.wgu[l]), T, 2 * cfg.ffn, d, 3, _ptr(self.act),
                             cfg.ffn, s))
            chk(lib.psk_gemm(_ptr(self.act), _ptr(w.wdown[l]), T, d, cfg.ffn, 2, _ptr(self.h), d, s))
