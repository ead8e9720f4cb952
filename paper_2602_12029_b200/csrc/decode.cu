// Decode-module step kernels: embedding, RMSNorm, grouped weight-streaming
// GEMV (K5), RoPE + paged KV append, shared-prefix paged decode attention
// (K6) and greedy argmax.
//
// Reference semantics: a decode module consumes the frozen base module's
// prompt KV for positions [0, n-1) and processes the last prompt token
// itself (frontend/src/model.ts:363-399, :372-374; evaluate.ts:16-19), then
// generates greedily one token per step (model.ts:388-399). The reference
// re-concatenates the whole past K/V every step (model.ts:307-310); here the
// KV is paged and appended in place, and one decode step of all co-batched
// modules reads each shared prompt page once.
#include "common.cuh"
#include "mma.cuh"

#include <math.h>
#include <stdlib.h>

namespace psk {
namespace dec {

constexpr int HD = 128;
constexpr int PT = 16;  // tokens per KV page (= kvstore block_size)

// ------------------------------------------------------------- embedding --

__global__ void embed_rows_kernel(psk_decode_batch b, const __nv_bfloat16* const* embed, int d,
                                  float* __restrict__ h) {
  pdl_wait();  // first kernel of a step: the previous step is fully done
  pdl_trigger();
  const int r = blockIdx.x;
  const __nv_bfloat16* row = embed[b.row_mod[r]] + (int64_t)b.tokens[r] * d;
  for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
    float f[8];
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(row + i), f);
    float4* o = reinterpret_cast<float4*>(h + (int64_t)r * d + i);
    o[0] = make_float4(f[0], f[1], f[2], f[3]);
    o[1] = make_float4(f[4], f[5], f[6], f[7]);
  }
}

// --------------------------------------------------------------- RMSNorm --

__global__ void rmsnorm_rows_kernel(const float* __restrict__ h, int d,
                                    const __nv_bfloat16* const* gamma, const int32_t* row_mod,
                                    float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float s_red[32];
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  const float* x = h + (int64_t)r * d;
  float ss = 0.f;
  for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(x + i);
    ss += v.x * v.x + v.y * v.y + v.z * v.z + v.w * v.w;
  }
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (blockDim.x >> 5) ? s_red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) s_red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(s_red[0] / (float)d + eps);
  const __nv_bfloat16* g = gamma[row_mod ? row_mod[r] : 0];
  __nv_bfloat16* o = out + (int64_t)r * d;
  for (int i = threadIdx.x * 4; i < d; i += blockDim.x * 4) {
    float4 v = *reinterpret_cast<const float4*>(x + i);
    __nv_bfloat162 g01 = *reinterpret_cast<const __nv_bfloat162*>(g + i);
    __nv_bfloat162 g23 = *reinterpret_cast<const __nv_bfloat162*>(g + i + 2);
    float2 a = __bfloat1622float2(g01), c = __bfloat1622float2(g23);
    __nv_bfloat162 o01 = __floats2bfloat162_rn(v.x * inv * a.x, v.y * inv * a.y);
    __nv_bfloat162 o23 = __floats2bfloat162_rn(v.z * inv * c.x, v.w * inv * c.y);
    *reinterpret_cast<__nv_bfloat162*>(o + i) = o01;
    *reinterpret_cast<__nv_bfloat162*>(o + i + 2) = o23;
  }
}

// ------------------------------------------------------------------ GEMV --
// Persistent, deterministic weight-streaming GEMV. The (module, row) space
// is cut into contiguous, `align`-row-aligned CTA ranges of near-equal size
// (so a 4-module QKV step spreads its 4 x 50 MB of weights over every SM);
// inside a CTA each warp takes a contiguous run of (row, 1024-element chunk)
// units, streams 4 x 16 B of W per lane per unit with L1-bypassing loads and
// keeps the few activation rows of that module in L1. Partials land in
// fixed shared-memory slots (no atomics) and are summed in a fixed order,
// so results are bit-reproducible run to run.
constexpr int GEMV_THREADS = 256;
#ifndef PSK_GEMV_V
#define PSK_GEMV_V 4
#endif
#ifndef PSK_GEMV_CTAS
#define PSK_GEMV_CTAS 3
#endif
#ifndef PSK_GEMV_PIPE
#define PSK_GEMV_PIPE 1
#endif
constexpr int GEMV_V = PSK_GEMV_V;         // 16-byte loads per lane per unit
constexpr int GEMV_CH = 32 * 8 * GEMV_V;   // elements per unit (1024)

template <int MAXM, int EPI>
__global__ void __launch_bounds__(GEMV_THREADS, PSK_GEMV_CTAS) gemv_kernel(  // one resident wave
    const __nv_bfloat16* __restrict__ X, int K, const __nv_bfloat16* const* W,
    const int32_t* __restrict__ mrs, int n_mod, int N, int align, void* out) {
  extern __shared__ float slots[];  // [rows_cta][cpr][MAXM]
  const int cpr = (K + GEMV_CH - 1) / GEMV_CH;
  const int64_t G = (int64_t)n_mod * N;
  const int64_t ngroups = G / align;
  const int64_t g0 = ((int64_t)blockIdx.x * ngroups / gridDim.x) * align;
  const int64_t g1 = ((int64_t)(blockIdx.x + 1) * ngroups / gridDim.x) * align;
  const int rows = (int)(g1 - g0);
  pdl_trigger();
  if (rows <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = GEMV_THREADS / 32;
  const int64_t units = (int64_t)rows * cpr;
  const int64_t u0 = warp * units / nw, u1 = (warp + 1) * units / nw;

  float acc[MAXM];
#pragma unroll
  for (int m = 0; m < MAXM; ++m) acc[m] = 0.f;
  int cur_row = -1, cur_slot = 0, M = 0, xbase = 0;

  // (a macro, not a by-reference lambda: that would put acc[] in local memory)
#define GEMV_FLUSH()                                                                   \
  if (cur_row >= 0) {                                                                  \
    _Pragma("unroll") for (int m = 0; m < MAXM; ++m) {                                 \
      float v = warp_sum(acc[m]);                                                      \
      if (lane == 0 && m < M) slots[((int64_t)cur_row * cpr + cur_slot) * MAXM + m] = v; \
      acc[m] = 0.f;                                                                    \
    }                                                                                  \
  }

  // zero all slots first (rows whose chunks are split over warps use only
  // the first chunk slot of each warp's run)
  for (int i = threadIdx.x; i < rows * cpr * MAXM; i += GEMV_THREADS) slots[i] = 0.f;
  __syncthreads();

  // Software pipeline: the weight loads of unit u+1 are issued before the
  // FMAs of unit u, so each lane keeps 2 x GEMV_V x 16 B of HBM reads in flight.
  uint4 wn[GEMV_V];
  int n_rl = 0, n_ch = 0, n_M = 0, n_xb = 0;
#define GEMV_FETCH(UU)                                                          \
  {                                                                             \
    n_rl = (int)((UU) / cpr);                                                   \
    n_ch = (int)((UU) % cpr);                                                   \
    const int64_t g_ = g0 + n_rl;                                               \
    const int mod_ = (int)(g_ / N);                                             \
    n_xb = mrs[mod_];                                                           \
    n_M = mrs[mod_ + 1] - n_xb;                                                 \
    const __nv_bfloat16* wr_ = W[mod_] + (int64_t)(g_ % N) * K;                 \
    _Pragma("unroll") for (int j = 0; j < GEMV_V; ++j) {                        \
      const int k = n_ch * GEMV_CH + j * 256 + lane * 8;                        \
      wn[j] = (n_M > 0 && k < K) ? ld_stream_v4(wr_ + k) : make_uint4(0, 0, 0, 0); \
    }                                                                           \
  }
  // the first weight unit streams while the producer of X drains (PDL)
  if (PSK_GEMV_PIPE && u0 < u1) GEMV_FETCH(u0);
  pdl_wait();
  for (int64_t u = u0; u < u1; ++u) {
    if (!PSK_GEMV_PIPE) GEMV_FETCH(u);
    uint4 w[GEMV_V];
#pragma unroll
    for (int j = 0; j < GEMV_V; ++j) w[j] = wn[j];
    const int rl = n_rl, ch = n_ch, uM = n_M, uxb = n_xb;
    if (PSK_GEMV_PIPE && u + 1 < u1) GEMV_FETCH(u + 1);
    if (rl != cur_row) {
      GEMV_FLUSH();
      cur_row = rl;
      cur_slot = ch;
      xbase = uxb;
      M = uM;
    }
    if (M == 0) continue;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      if (m < M) {
        const __nv_bfloat16* xr = X + (int64_t)(xbase + m) * K;
#pragma unroll
        for (int j = 0; j < GEMV_V; ++j) {
          const int k = ch * GEMV_CH + j * 256 + lane * 8;
          if (k < K) {
            uint4 xv = __ldg(reinterpret_cast<const uint4*>(xr + k));
            float wf[8], xf[8];
            bf16x8_to_f32(w[j], wf);
            bf16x8_to_f32(xv, xf);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[m] = fmaf(wf[e], xf[e], acc[m]);
          }
        }
      }
    }
  }
  GEMV_FLUSH();
#undef GEMV_FLUSH
#undef GEMV_FETCH
  __syncthreads();

  // epilogue: thread per (row, m)
  if (EPI == PSK_EPI_SILU_MUL) {
    // rows come in groups of 32: [gate 16 | up 16] -> 16 outputs
    const int pairs = rows / 2;
    for (int i = threadIdx.x; i < pairs * MAXM; i += GEMV_THREADS) {
      const int pi = i / MAXM, m = i % MAXM;
      const int grp = pi / 16, lo = pi % 16;
      const int rg = grp * 32 + lo, ru = rg + 16;
      const int64_t gg = g0 + rg;
      const int mod = (int)(gg / N);
      const int n = (int)(gg % N);
      const int Mm = mrs[mod + 1] - mrs[mod];
      if (m >= Mm) continue;
      float vg = 0.f, vu = 0.f;
      for (int c = 0; c < cpr; ++c) {
        vg += slots[((int64_t)rg * cpr + c) * MAXM + m];
        vu += slots[((int64_t)ru * cpr + c) * MAXM + m];
      }
      const float s = vg / (1.f + __expf(-vg));
      const int f = (n / 32) * 16 + (n % 16);
      reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)(mrs[mod] + m) * (N / 2) + f] = f2bf(s * vu);
    }
  } else {
    for (int i = threadIdx.x; i < rows * MAXM; i += GEMV_THREADS) {
      const int rl = i / MAXM, m = i % MAXM;
      const int64_t gg = g0 + rl;
      const int mod = (int)(gg / N);
      const int n = (int)(gg % N);
      const int Mm = mrs[mod + 1] - mrs[mod];
      if (m >= Mm) continue;
      float v = 0.f;
      for (int c = 0; c < cpr; ++c) v += slots[((int64_t)rl * cpr + c) * MAXM + m];
      const int64_t o = (int64_t)(mrs[mod] + m) * N + n;
      if (EPI == PSK_EPI_STORE_BF16) reinterpret_cast<__nv_bfloat16*>(out)[o] = f2bf(v);
      if (EPI == PSK_EPI_STORE_F32) reinterpret_cast<float*>(out)[o] = v;
      if (EPI == PSK_EPI_RESID_ADD) reinterpret_cast<float*>(out)[o] += v;
    }
  }
}

// -------------------------------------------------- tensor-core GEMV ----
// For 2..16 rows per module (multi-session decode batches) the FMA count per
// weight byte outgrows the CUDA cores, so the dot products run on mma.sync
// m16n8k16 (W = A operand, 16 weight rows; x = B operand, 8 activation rows
// per n-tile). Weights are still streamed straight from HBM into registers:
// a fixed permutation of k inside every 32-column chunk (applied identically
// to W and x; a dot product is permutation-invariant) makes thread t of a
// quad own physical columns [8t, 8t+8) = its A/B fragments for two k-steps,
// so every fragment is one coalesced 16-byte load. Work unit = (16-row tile,
// 1024-column chunk); each unit's partial lands in its own shared-memory
// slot (deterministic, no atomics) and the epilogue is the scalar one above.
template <int NT, int EPI>
__global__ void __launch_bounds__(GEMV_THREADS, PSK_GEMV_CTAS) gemv_mma_kernel(
    const __nv_bfloat16* __restrict__ X, int K, const __nv_bfloat16* const* W,
    const int32_t* __restrict__ mrs, int n_mod, int N, int align, void* out) {
  constexpr int MAXM = NT * 8;
  extern __shared__ float slots[];  // [rows_cta][cpr][MAXM]
  const int cpr = (K + GEMV_CH - 1) / GEMV_CH;
  const int64_t G = (int64_t)n_mod * N;
  const int64_t ngroups = G / align;
  const int64_t g0 = ((int64_t)blockIdx.x * ngroups / gridDim.x) * align;
  const int64_t g1 = ((int64_t)(blockIdx.x + 1) * ngroups / gridDim.x) * align;
  const int rows = (int)(g1 - g0);
  pdl_trigger();
  if (rows <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int tiles = rows / 16;
  const int64_t units = (int64_t)tiles * cpr;
  const int64_t u0 = warp * units / (GEMV_THREADS / 32), u1 = (warp + 1) * units / (GEMV_THREADS / 32);
  for (int i = threadIdx.x; i < rows * cpr * MAXM; i += GEMV_THREADS) slots[i] = 0.f;
  __syncthreads();
  pdl_wait();
  for (int64_t u = u0; u < u1; ++u) {
    const int tl = (int)(u / cpr), ch = (int)(u % cpr);
    const int64_t r0 = g0 + (int64_t)tl * 16;
    const int mod = (int)(r0 / N);
    const int xb = mrs[mod], M = mrs[mod + 1] - xb;
    if (M == 0) continue;
    const __nv_bfloat16* wa_p = W[mod] + (r0 % N + gq) * (int64_t)K;
    const __nv_bfloat16* wb_p = wa_p + 8 * (int64_t)K;
    float c[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[nt][0] = c[nt][1] = c[nt][2] = c[nt][3] = 0.f;
    const int cbeg = ch * GEMV_CH + tq * 8;
    const int cend = min(K, (ch + 1) * GEMV_CH);
#pragma unroll 1
    for (int col0 = cbeg; col0 < cend; col0 += 4 * 32) {
      uint4 wa[4], wb[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = col0 + q * 32;
        const bool ok = col < cend;
        wa[q] = ok ? ld_stream_v4(wa_p + col) : make_uint4(0, 0, 0, 0);
        wb[q] = ok ? ld_stream_v4(wb_p + col) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int col = col0 + q * 32;
        if (col >= cend) break;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int xr = nt * 8 + gq;
          const uint4 xv = xr < M ? __ldg(reinterpret_cast<const uint4*>(X + (int64_t)(xb + xr) * K + col))
                                  : make_uint4(0, 0, 0, 0);
          const uint32_t a0[4] = {wa[q].x, wb[q].x, wa[q].y, wb[q].y};
          const uint32_t a1[4] = {wa[q].z, wb[q].z, wa[q].w, wb[q].w};
          mma_bf16_16816(c[nt], a0, xv.x, xv.y);
          mma_bf16_16816(c[nt], a1, xv.z, xv.w);
        }
      }
    }
    // C fragment: (row gq / gq+8, cols 2tq, 2tq+1) of [16 weight rows x 8 x rows]
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int m = nt * 8 + 2 * tq;
      float* s0 = slots + ((int64_t)(tl * 16 + gq) * cpr + ch) * MAXM;
      float* s8 = slots + ((int64_t)(tl * 16 + gq + 8) * cpr + ch) * MAXM;
      if (m < M) { s0[m] = c[nt][0]; s8[m] = c[nt][2]; }
      if (m + 1 < M) { s0[m + 1] = c[nt][1]; s8[m + 1] = c[nt][3]; }
    }
  }
  __syncthreads();
  if (EPI == PSK_EPI_SILU_MUL) {
    const int pairs = rows / 2;
    for (int i = threadIdx.x; i < pairs * MAXM; i += GEMV_THREADS) {
      const int pi = i / MAXM, m = i % MAXM;
      const int rg = (pi / 16) * 32 + pi % 16, ru = rg + 16;
      const int64_t gg = g0 + rg;
      const int mod = (int)(gg / N);
      const int n = (int)(gg % N);
      if (m >= mrs[mod + 1] - mrs[mod]) continue;
      float vg = 0.f, vu = 0.f;
      for (int cc = 0; cc < cpr; ++cc) {
        vg += slots[((int64_t)rg * cpr + cc) * MAXM + m];
        vu += slots[((int64_t)ru * cpr + cc) * MAXM + m];
      }
      const float sg = vg / (1.f + __expf(-vg));
      reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)(mrs[mod] + m) * (N / 2) + (n / 32) * 16 + n % 16] =
          f2bf(sg * vu);
    }
  } else {
    for (int i = threadIdx.x; i < rows * MAXM; i += GEMV_THREADS) {
      const int rl = i / MAXM, m = i % MAXM;
      const int64_t gg = g0 + rl;
      const int mod = (int)(gg / N);
      const int n = (int)(gg % N);
      if (m >= mrs[mod + 1] - mrs[mod]) continue;
      float v = 0.f;
      for (int cc = 0; cc < cpr; ++cc) v += slots[((int64_t)rl * cpr + cc) * MAXM + m];
      const int64_t o = (int64_t)(mrs[mod] + m) * N + n;
      if (EPI == PSK_EPI_STORE_BF16) reinterpret_cast<__nv_bfloat16*>(out)[o] = f2bf(v);
      if (EPI == PSK_EPI_STORE_F32) reinterpret_cast<float*>(out)[o] = v;
      if (EPI == PSK_EPI_RESID_ADD) reinterpret_cast<float*>(out)[o] += v;
    }
  }
}

// ---------------------------------------------------- RoPE + KV append ---

__device__ __forceinline__ __nv_bfloat16* kv_ptr(const psk_kv_layout& kv, int32_t page, int layer,
                                                 int kvsel, int head, int tok) {
  return reinterpret_cast<__nv_bfloat16*>(kv.base) + (int64_t)page * kv.page_elems +
         ((((int64_t)layer * 2 + kvsel) * kv.n_kv_heads + head) * kv.page_tokens + tok) * kv.head_dim;
}

__global__ void rope_append_kernel(psk_decode_batch b, const float* __restrict__ qkv, int nq,
                                   const float* __restrict__ rope, int layer, psk_kv_layout kv,
                                   __nv_bfloat16* __restrict__ q_rot) {
  // the attention kernel (PDL-launched next) may start its table prologue now
  asm volatile("griddepcontrol.launch_dependents;");
  const int r = blockIdx.x;
  const int nkv = kv.n_kv_heads;
  const int idx = b.priv_len[r];
  const int pos = b.sess_len[b.row_sess[r]] + idx;
  const int page = b.row_pages[(int64_t)r * b.max_row_pages + idx / PT];
  const int off = idx % PT;
  const float* row = qkv + (int64_t)r * (nq + 2 * nkv) * HD;
  const float* cs = rope + (int64_t)pos * HD;  // [64][2]
  const int i = threadIdx.x;                    // 0..63
  const float c = cs[2 * i], s = cs[2 * i + 1];
  pdl_wait();  // qkv comes from the GEMV just before
  for (int h = 0; h < nq; ++h) {
    const float x1 = row[h * HD + i], x2 = row[h * HD + i + 64];
    q_rot[((int64_t)r * nq + h) * HD + i] = f2bf(x1 * c - x2 * s);
    q_rot[((int64_t)r * nq + h) * HD + i + 64] = f2bf(x2 * c + x1 * s);
  }
  for (int h = 0; h < nkv; ++h) {
    const float* kr = row + (nq + h) * HD;
    const float* vr = row + (nq + nkv + h) * HD;
    __nv_bfloat16* kd = kv_ptr(kv, page, layer, 0, h, off);
    __nv_bfloat16* vd = kv_ptr(kv, page, layer, 1, h, off);
    const float x1 = kr[i], x2 = kr[i + 64];
    kd[i] = f2bf(x1 * c - x2 * s);
    kd[i + 64] = f2bf(x2 * c + x1 * s);
    vd[i] = f2bf(vr[i]);
    vd[i + 64] = f2bf(vr[i + 64]);
  }
}

// ---------------------------------------------------------------- argmax --

__global__ void argmax_advance_kernel(psk_decode_batch b, const float* __restrict__ logits, int V,
                                      int32_t* __restrict__ out_tokens, int max_new) {
  __shared__ float s_v[32];
  __shared__ int s_i[32];
  pdl_wait();
  const int r = blockIdx.x;
  const float* x = logits + (int64_t)r * V;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  for (int i = threadIdx.x; i < V; i += blockDim.x) {
    const float v = x[i];
    if (v > bv) { bv = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { s_v[threadIdx.x >> 5] = bv; s_i[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x < 32) {
    const int nw = blockDim.x >> 5;
    bv = threadIdx.x < nw ? s_v[threadIdx.x] : -INFINITY;
    bi = threadIdx.x < nw ? s_i[threadIdx.x] : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if (threadIdx.x == 0) {
      const int k = b.priv_len[r];
      if (out_tokens && k < max_new) out_tokens[(int64_t)r * max_new + k] = bi;
      b.tokens[r] = bi;
      // saturate at the row's page capacity: idle continuous-batching slots keep
      // stepping without ever indexing past their private page table
      b.priv_len[r] = min(k + 1, b.max_row_pages * PT - 1);
    }
  }
}

}  // namespace dec
}  // namespace psk

using namespace psk::dec;

namespace {

template <int MAXM, bool MMA = false>
int launch_gemv(const void* x, int K, const void* const* W, const int32_t* mrs, int n_mod, int N,
                int epi, void* out, cudaStream_t s) {
  const int align = epi == PSK_EPI_SILU_MUL ? 32 : (MMA ? 16 : 1);
  const int cpr = (K + GEMV_CH - 1) / GEMV_CH;
  const int64_t G = (int64_t)n_mod * N;
  static int sms = 0;
  if (!sms) {
    int dev;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  int grid = sms * PSK_GEMV_CTAS;  // one resident wave (matches the launch bounds)
  // keep the partial slots of PSK_GEMV_CTAS co-resident CTAs within shared memory
  const int64_t slot_bytes_per_row = (int64_t)cpr * MAXM * 4;
  const int64_t smem_cap = (225 * 1024) / PSK_GEMV_CTAS;
  while (((G + grid - 1) / grid + align) * slot_bytes_per_row > smem_cap) grid += sms;
  if (grid > G / align) grid = (int)(G / align);
  const size_t smem = (size_t)(((G / align + grid - 1) / grid) * align) * slot_bytes_per_row;
  auto xb = reinterpret_cast<const __nv_bfloat16*>(x);
  auto Wb = reinterpret_cast<const __nv_bfloat16* const*>(W);
#define PSK_GEMV_CASE(E)                                                                        \
  case E: {                                                                                     \
    auto k = MMA ? gemv_mma_kernel<(MAXM + 7) / 8, E> : gemv_kernel<MAXM, E>;                   \
    if (smem > 48 * 1024)                                                                       \
      PSK_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    PSK_CUDA_TRY(psk::launch_pdl(k, dim3(grid), dim3(GEMV_THREADS), smem, s, xb, K, Wb, mrs,   \
                                 n_mod, N, align, out));                                        \
    break;                                                                                      \
  }
  switch (epi) {
    PSK_GEMV_CASE(PSK_EPI_STORE_BF16)
    PSK_GEMV_CASE(PSK_EPI_STORE_F32)
    PSK_GEMV_CASE(PSK_EPI_RESID_ADD)
    PSK_GEMV_CASE(PSK_EPI_SILU_MUL)
    default:
      psk::set_error("psk_gemv: unknown epilogue %d", epi);
      return PSK_EINVAL;
  }
#undef PSK_GEMV_CASE
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // namespace

extern "C" {

int psk_embed_rows(const psk_decode_batch* b, const void* const* embed, int32_t d, float* h,
                   void* stream) {
  PSK_CHECK_ARG(b && embed && h && d % 8 == 0, "psk_embed_rows: bad args");
  if (b->n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(embed_rows_kernel, dim3(b->n_rows), dim3(128), 0, psk::as_stream(stream),
                               *b, reinterpret_cast<const __nv_bfloat16* const*>(embed), d, h));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_rmsnorm_rows(const float* h, int32_t n_rows, int32_t d, const void* const* gamma,
                     const int32_t* row_mod, float eps, void* out, void* stream) {
  PSK_CHECK_ARG(h && gamma && out && d % 4 == 0 && n_rows >= 0, "psk_rmsnorm_rows: bad args");
  if (n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(rmsnorm_rows_kernel, dim3(n_rows), dim3(256), 0, psk::as_stream(stream),
                               h, d, reinterpret_cast<const __nv_bfloat16* const*>(gamma), row_mod,
                               eps, reinterpret_cast<__nv_bfloat16*>(out)));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_gemv(const void* x, int32_t n_rows, int32_t K, const void* const* W,
             const int32_t* mod_row_start, int32_t n_mod, int32_t N, int32_t epilogue, void* out,
             void* stream) {
  PSK_CHECK_ARG(x && W && mod_row_start && out && K % 8 == 0 && N > 0 && n_mod > 0,
                "psk_gemv: bad args");
  PSK_CHECK_ARG(epilogue != PSK_EPI_SILU_MUL || N % 32 == 0, "psk_gemv: SILU_MUL needs N%%32==0");
  const int maxm = n_rows - n_mod + 1;
  cudaStream_t s = psk::as_stream(stream);
  if (maxm <= 1) return launch_gemv<1>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
  if (N % 16 == 0 && !getenv("PSK_GEMV_SCALAR")) {  // tensor-core path for 2..16 rows / module
    if (maxm <= 8) return launch_gemv<8, true>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
    if (maxm <= 16) return launch_gemv<16, true>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
  }
  if (maxm <= 2) return launch_gemv<2>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
  if (maxm <= 4) return launch_gemv<4>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
  if (maxm <= 8) return launch_gemv<8>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
  if (maxm <= 16) return launch_gemv<16>(x, K, W, mod_row_start, n_mod, N, epilogue, out, s);
  psk::set_error("psk_gemv: more than 16 rows per module (%d)", maxm);
  return PSK_EINVAL;
}

int psk_rope_append(const psk_decode_batch* b, const float* qkv, int32_t n_q_heads,
                    const float* rope, int32_t layer, psk_kv_layout kv, void* q_rot, void* stream) {
  PSK_CHECK_ARG(b && qkv && rope && q_rot && kv.head_dim == HD && kv.page_tokens == PT,
                "psk_rope_append: bad args (head_dim must be 128, page_tokens 16)");
  if (b->n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(rope_append_kernel, dim3(b->n_rows), dim3(64), 0, psk::as_stream(stream),
                               *b, qkv, n_q_heads, rope, layer, kv,
                               reinterpret_cast<__nv_bfloat16*>(q_rot)));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_argmax_advance(const psk_decode_batch* b, const float* logits, int32_t vocab,
                       int32_t* out_tokens, int32_t max_new, void* stream) {
  PSK_CHECK_ARG(b && logits && vocab > 0, "psk_argmax_advance: bad args");
  if (b->n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(argmax_advance_kernel, dim3(b->n_rows), dim3(1024), 0,
                               psk::as_stream(stream), *b, logits, vocab, out_tokens, max_new));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // extern "C"
