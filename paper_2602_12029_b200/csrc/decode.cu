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

namespace psk {
namespace dec {

constexpr int HD = 128;
constexpr int PT = 16;  // tokens per KV page (= kvstore block_size)

// ------------------------------------------------------------- embedding --

__global__ void embed_rows_kernel(psk_decode_batch b, const __nv_bfloat16* const* embed, int d,
                                  float* __restrict__ h) {
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
constexpr int GEMV_V = 4;                  // 16-byte loads per lane per unit
constexpr int GEMV_CH = 32 * 8 * GEMV_V;   // elements per unit (1024)

template <int MAXM, int EPI>
__global__ void __launch_bounds__(GEMV_THREADS) gemv_kernel(
    const __nv_bfloat16* __restrict__ X, int K, const __nv_bfloat16* const* W,
    const int32_t* __restrict__ mrs, int n_mod, int N, int align, void* out) {
  extern __shared__ float slots[];  // [rows_cta][cpr][MAXM]
  const int cpr = (K + GEMV_CH - 1) / GEMV_CH;
  const int64_t G = (int64_t)n_mod * N;
  const int64_t ngroups = G / align;
  const int64_t g0 = ((int64_t)blockIdx.x * ngroups / gridDim.x) * align;
  const int64_t g1 = ((int64_t)(blockIdx.x + 1) * ngroups / gridDim.x) * align;
  const int rows = (int)(g1 - g0);
  if (rows <= 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = GEMV_THREADS / 32;
  const int64_t units = (int64_t)rows * cpr;
  const int64_t u0 = warp * units / nw, u1 = (warp + 1) * units / nw;

  float acc[MAXM];
#pragma unroll
  for (int m = 0; m < MAXM; ++m) acc[m] = 0.f;
  int cur_row = -1, cur_slot = 0, M = 0, xbase = 0;
  const __nv_bfloat16* wrow = nullptr;

  auto flush = [&]() {
    if (cur_row < 0) return;
#pragma unroll
    for (int m = 0; m < MAXM; ++m) {
      float v = warp_sum(acc[m]);
      if (lane == 0 && m < M) slots[((int64_t)cur_row * cpr + cur_slot) * MAXM + m] = v;
      acc[m] = 0.f;
    }
  };

  // zero all slots first (rows whose chunks are split over warps use only
  // the first chunk slot of each warp's run)
  for (int i = threadIdx.x; i < rows * cpr * MAXM; i += GEMV_THREADS) slots[i] = 0.f;
  __syncthreads();

  for (int64_t u = u0; u < u1; ++u) {
    const int rl = (int)(u / cpr);
    const int ch = (int)(u % cpr);
    if (rl != cur_row) {
      flush();
      cur_row = rl;
      cur_slot = ch;
      const int64_t g = g0 + rl;
      const int mod = (int)(g / N);
      const int n = (int)(g % N);
      xbase = mrs[mod];
      M = mrs[mod + 1] - xbase;
      wrow = W[mod] + (int64_t)n * K;
    }
    if (M == 0) continue;
    uint4 w[GEMV_V];
#pragma unroll
    for (int j = 0; j < GEMV_V; ++j) {
      const int k = ch * GEMV_CH + j * 256 + lane * 8;
      w[j] = k < K ? ld_stream_v4(wrow + k) : make_uint4(0, 0, 0, 0);
    }
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
  flush();
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

// ---------------------------------------------------- RoPE + KV append ---

__device__ __forceinline__ __nv_bfloat16* kv_ptr(const psk_kv_layout& kv, int32_t page, int layer,
                                                 int kvsel, int head, int tok) {
  return reinterpret_cast<__nv_bfloat16*>(kv.base) + (int64_t)page * kv.page_elems +
         ((((int64_t)layer * 2 + kvsel) * kv.n_kv_heads + head) * kv.page_tokens + tok) * kv.head_dim;
}

__global__ void rope_append_kernel(psk_decode_batch b, const float* __restrict__ qkv, int nq,
                                   const float* __restrict__ rope, int layer, psk_kv_layout kv,
                                   __nv_bfloat16* __restrict__ q_rot) {
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

// ------------------------------------------------------ decode attention --
// One CTA = (session | row, kv head, split). 4 warps. The CTA streams its
// pages (K and V 4 KiB tiles) through a 3-stage cp.async ring of 4-page
// rounds into XOR-swizzled shared memory; warps map to (query m-tile, page
// subset) so every page is read from HBM once and consumed by all query
// rows of the session: GQA group x co-batched decode modules, up to 64 rows.
constexpr int AT_WARPS = 4;
constexpr int AT_THREADS = AT_WARPS * 32;
constexpr int AT_RP = 4;      // pages per round
constexpr int AT_NST = 3;     // pipeline stages
constexpr int AT_TILE = PT * HD * 2;  // bytes per K (or V) tile: 4 KiB
constexpr int AT_STAGE = AT_RP * 2 * AT_TILE;
constexpr int AT_SMEM = AT_NST * AT_STAGE;  // 96 KiB
constexpr int AT_GMAX = 64;

struct AttnParams {
  psk_decode_batch b;
  psk_kv_layout kv;
  const __nv_bfloat16* q;  // [rows][nq][HD]
  int nq, grp, layer;
  int ns_shared, ns_priv;
  int n_shared_items;
  int gstride;   // query slots per item in the workspace
  float* pm;     // [items][gstride]
  float* pl;
  float* po;     // [items][gstride][HD]
  float scale_log2;
};

__global__ void __launch_bounds__(AT_THREADS, 2) decode_attn_partial_kernel(AttnParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  int item = blockIdx.x;
  bool shared_item = item < p.n_shared_items;
  int h, j, L, G, ns;
  const int32_t* table;
  int sess = -1, row = -1;
  if (shared_item) {
    ns = p.ns_shared;
    sess = item / (nkv * ns);
    h = (item / ns) % nkv;
    j = item % ns;
    L = p.b.sess_len[sess];
    G = p.b.sess_nrows[sess] * p.grp;
    table = p.b.sess_pages + (int64_t)sess * p.b.max_sess_pages;
  } else {
    const int it = item - p.n_shared_items;
    ns = p.ns_priv;
    row = it / (nkv * ns);
    h = (it / ns) % nkv;
    j = it % ns;
    L = p.b.priv_len[row] + 1;  // includes the token appended this step
    G = p.grp;
    table = p.b.row_pages + (int64_t)row * p.b.max_row_pages;
  }
  const int P = (L + PT - 1) / PT;
  const int pb = (int)((int64_t)j * P / ns), pe = (int)((int64_t)(j + 1) * P / ns);
  const int tiles = (G + 15) / 16;
  const int ways = tiles <= 1 ? 4 : (tiles == 2 ? 2 : 1);
  const int my_tile = warp / ways;
  const int my_way = warp % ways;
  const bool active = my_tile < tiles;

  // -- query fragments for my m-tile (A operand, 8 k-steps)
  uint32_t qa[8][4];
  {
    const int gA = my_tile * 16 + (lane >> 2), gB = gA + 8;
    const int t2 = (lane & 3) * 2;
    auto qrow = [&](int g) -> const __nv_bfloat16* {
      if (!active || g >= G) return nullptr;
      int qr, qh;
      if (shared_item) {
        qr = p.b.sess_rows[(int64_t)sess * p.b.max_rows_per_sess + g / p.grp];
        qh = h * p.grp + g % p.grp;
      } else {
        qr = row;
        qh = h * p.grp + g;
      }
      return p.q + ((int64_t)qr * p.nq + qh) * HD;
    };
    const __nv_bfloat16* qA = qrow(gA);
    const __nv_bfloat16* qB = qrow(gB);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c0 = ks * 16 + t2, c1 = c0 + 8;
      qa[ks][0] = qA ? *reinterpret_cast<const uint32_t*>(qA + c0) : 0u;
      qa[ks][1] = qB ? *reinterpret_cast<const uint32_t*>(qB + c0) : 0u;
      qa[ks][2] = qA ? *reinterpret_cast<const uint32_t*>(qA + c1) : 0u;
      qa[ks][3] = qB ? *reinterpret_cast<const uint32_t*>(qB + c1) : 0u;
    }
  }

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const int rounds = (pe - pb + AT_RP - 1) / AT_RP;
  const uint32_t sbase = smem_u32(smem);
  auto issue = [&](int rd) {
    if (rd < rounds) {
      const uint32_t st = sbase + (rd % AT_NST) * AT_STAGE;
      for (int e = threadIdx.x; e < AT_RP * 2 * 256; e += AT_THREADS) {
        const int pslot = e >> 9, kvsel = (e >> 8) & 1, ce = e & 255;
        const int pg = pb + rd * AT_RP + pslot;
        if (pg < pe) {
          const int page = table[pg];
          const __nv_bfloat16* src = kv_ptr(p.kv, page, p.layer, kvsel, h, 0);
          const int tr = ce >> 4, c = ce & 15;
          cp_async16(st + (pslot * 2 + kvsel) * AT_TILE + swz256(tr, c), src + tr * HD + c * 8);
        }
      }
    }
    cp_async_commit();
  };

#pragma unroll
  for (int s = 0; s < AT_NST - 1; ++s) issue(s);

  for (int rd = 0; rd < rounds; ++rd) {
    cp_async_wait<AT_NST - 2>();
    __syncthreads();
    issue(rd + AT_NST - 1);
    if (active) {
      const uint32_t st = sbase + (rd % AT_NST) * AT_STAGE;
      for (int pslot = my_way; pslot < AT_RP; pslot += ways) {
        const int pg = pb + rd * AT_RP + pslot;
        if (pg >= pe) break;
        const uint32_t kt = st + (pslot * 2 + 0) * AT_TILE;
        const uint32_t vt = st + (pslot * 2 + 1) * AT_TILE;
        float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
        {
          const int mi = lane >> 3, ri = lane & 7;
          const int tok = (mi >> 1) * 8 + ri;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            uint32_t b0, b1, b2, b3;
            ldmatrix_x4(kt + swz256(tok, 2 * ks + (mi & 1)), b0, b1, b2, b3);
            mma_bf16_16816(s[0], qa[ks], b0, b1);
            mma_bf16_16816(s[1], qa[ks], b2, b3);
          }
        }
        // scale + mask (tokens past L in the last page)
        const int tok0 = pg * PT;
        const int cb = (lane & 3) * 2;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int t = tok0 + nt * 8 + cb + (e & 1);
            s[nt][e] = t < L ? s[nt][e] * p.scale_log2 : -INFINITY;
          }
        float mx0 = fmaxf(fmaxf(s[0][0], s[0][1]), fmaxf(s[1][0], s[1][1]));
        float mx1 = fmaxf(fmaxf(s[0][2], s[0][3]), fmaxf(s[1][2], s[1][3]));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
        const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
        const float r0 = n0 == -INFINITY ? 0.f : n0, r1 = n1 == -INFINITY ? 0.f : n1;
        const float c0 = exp2f(m0 - r0), c1 = exp2f(m1 - r1);
        m0 = n0;
        m1 = n1;
        float pr[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          pr[nt][0] = exp2f(s[nt][0] - r0);
          pr[nt][1] = exp2f(s[nt][1] - r0);
          pr[nt][2] = exp2f(s[nt][2] - r1);
          pr[nt][3] = exp2f(s[nt][3] - r1);
        }
        l0 = l0 * c0 + pr[0][0] + pr[0][1] + pr[1][0] + pr[1][1];
        l1 = l1 * c1 + pr[0][2] + pr[0][3] + pr[1][2] + pr[1][3];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          o[i][0] *= c0;
          o[i][1] *= c0;
          o[i][2] *= c1;
          o[i][3] *= c1;
        }
        uint32_t pa[4];
        pa[0] = pack_bf16(pr[0][0], pr[0][1]);
        pa[1] = pack_bf16(pr[0][2], pr[0][3]);
        pa[2] = pack_bf16(pr[1][0], pr[1][1]);
        pa[3] = pack_bf16(pr[1][2], pr[1][3]);
        {
          const int mi = lane >> 3, ri = lane & 7;
          const int tok = (mi & 1) * 8 + ri;
#pragma unroll
          for (int np = 0; np < 8; ++np) {
            uint32_t b0, b1, b2, b3;
            ldmatrix_x4_trans(vt + swz256(tok, 2 * np + (mi >> 1)), b0, b1, b2, b3);
            mma_bf16_16816(o[2 * np], pa, b0, b1);
            mma_bf16_16816(o[2 * np + 1], pa, b2, b3);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();

  // -- combine the `ways` warps of each m-tile through shared memory
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  float* sO = reinterpret_cast<float*>(smem);              // [4 warps][16][HD]
  float* sM = sO + AT_WARPS * 16 * HD;                      // [4][16]
  float* sL = sM + AT_WARPS * 16;                           // [4][16]
  {
    const int ra = lane >> 2, rb = ra + 8, cb = (lane & 3) * 2;
    float* w = sO + warp * 16 * HD;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      w[ra * HD + nt * 8 + cb] = o[nt][0];
      w[ra * HD + nt * 8 + cb + 1] = o[nt][1];
      w[rb * HD + nt * 8 + cb] = o[nt][2];
      w[rb * HD + nt * 8 + cb + 1] = o[nt][3];
    }
    if ((lane & 3) == 0) {
      sM[warp * 16 + ra] = m0;
      sM[warp * 16 + rb] = m1;
      sL[warp * 16 + ra] = l0;
      sL[warp * 16 + rb] = l1;
    }
  }
  __syncthreads();
  const int64_t base_slot = (int64_t)item * p.gstride;
  for (int e = threadIdx.x; e < tiles * 16 * HD; e += AT_THREADS) {
    const int t = e / (16 * HD), rr = (e / HD) % 16, d = e % HD;
    const int g = t * 16 + rr;
    if (g >= G) continue;
    float M = -INFINITY;
    for (int w = 0; w < ways; ++w) M = fmaxf(M, sM[(t * ways + w) * 16 + rr]);
    const float Mr = M == -INFINITY ? 0.f : M;
    float acc = 0.f, lsum = 0.f;
    for (int w = 0; w < ways; ++w) {
      const int ww = t * ways + w;
      const float f = exp2f(sM[ww * 16 + rr] - Mr);
      acc += f * sO[(ww * 16 + rr) * HD + d];
      lsum += f * sL[ww * 16 + rr];
    }
    p.po[(base_slot + g) * HD + d] = acc;
    if (d == 0) {
      p.pm[base_slot + g] = M;
      p.pl[base_slot + g] = lsum;
    }
  }
}

__global__ void decode_attn_merge_kernel(AttnParams p, __nv_bfloat16* __restrict__ out) {
  const int r = blockIdx.x, qh = blockIdx.y, d = threadIdx.x;
  const int nkv = p.kv.n_kv_heads;
  const int h = qh / p.grp, ql = qh % p.grp;
  const int s = p.b.row_sess[r];
  const int gs = p.b.row_in_sess[r] * p.grp + ql;
  float M = -INFINITY;
  for (int j = 0; j < p.ns_shared; ++j)
    M = fmaxf(M, p.pm[((int64_t)(s * nkv + h) * p.ns_shared + j) * p.gstride + gs]);
  for (int j = 0; j < p.ns_priv; ++j)
    M = fmaxf(M, p.pm[((int64_t)p.n_shared_items + (r * nkv + h) * p.ns_priv + j) * p.gstride + ql]);
  const float Mr = M == -INFINITY ? 0.f : M;
  float acc = 0.f, lsum = 0.f;
  for (int j = 0; j < p.ns_shared; ++j) {
    const int64_t sl = ((int64_t)(s * nkv + h) * p.ns_shared + j) * p.gstride + gs;
    const float f = exp2f(p.pm[sl] - Mr);
    acc += f * p.po[sl * HD + d];
    lsum += f * p.pl[sl];
  }
  for (int j = 0; j < p.ns_priv; ++j) {
    const int64_t sl = ((int64_t)p.n_shared_items + (r * nkv + h) * p.ns_priv + j) * p.gstride + ql;
    const float f = exp2f(p.pm[sl] - Mr);
    acc += f * p.po[sl * HD + d];
    lsum += f * p.pl[sl];
  }
  out[((int64_t)r * p.nq + qh) * HD + d] = f2bf(acc / lsum);
}

// ---------------------------------------------------------------- argmax --

__global__ void argmax_advance_kernel(psk_decode_batch b, const float* __restrict__ logits, int V,
                                      int32_t* __restrict__ out_tokens, int max_new) {
  __shared__ float s_v[32];
  __shared__ int s_i[32];
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
      b.priv_len[r] = k + 1;
    }
  }
}

}  // namespace dec
}  // namespace psk

using namespace psk::dec;

namespace {

int attn_items(const psk_decode_batch* b, int nkv, int nss, int nsp, int* n_shared, int* n_total,
               int* gstride) {
  *n_shared = b->n_sess * nkv * nss;
  *n_total = *n_shared + b->n_rows * nkv * nsp;
  (void)gstride;
  return 0;
}

template <int MAXM>
int launch_gemv(const void* x, int K, const void* const* W, const int32_t* mrs, int n_mod, int N,
                int epi, void* out, cudaStream_t s) {
  const int align = epi == PSK_EPI_SILU_MUL ? 32 : 1;
  const int cpr = (K + GEMV_CH - 1) / GEMV_CH;
  const int64_t G = (int64_t)n_mod * N;
  int grid = 148 * 4;
  // keep the partial slots of one CTA within 64 KiB of shared memory
  const int64_t slot_bytes_per_row = (int64_t)cpr * MAXM * 4;
  while (((G + grid - 1) / grid + align) * slot_bytes_per_row > 64 * 1024) grid += 148;
  if (grid > G / align) grid = (int)(G / align);
  const size_t smem = (size_t)(((G / align + grid - 1) / grid) * align) * slot_bytes_per_row;
  auto xb = reinterpret_cast<const __nv_bfloat16*>(x);
  auto Wb = reinterpret_cast<const __nv_bfloat16* const*>(W);
#define PSK_GEMV_CASE(E)                                                                        \
  case E: {                                                                                     \
    auto k = gemv_kernel<MAXM, E>;                                                              \
    if (smem > 48 * 1024)                                                                       \
      PSK_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)); \
    k<<<grid, GEMV_THREADS, smem, s>>>(xb, K, Wb, mrs, n_mod, N, align, out);                  \
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
  embed_rows_kernel<<<b->n_rows, 128, 0, psk::as_stream(stream)>>>(
      *b, reinterpret_cast<const __nv_bfloat16* const*>(embed), d, h);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_rmsnorm_rows(const float* h, int32_t n_rows, int32_t d, const void* const* gamma,
                     const int32_t* row_mod, float eps, void* out, void* stream) {
  PSK_CHECK_ARG(h && gamma && out && d % 4 == 0 && n_rows >= 0, "psk_rmsnorm_rows: bad args");
  if (n_rows == 0) return PSK_OK;
  rmsnorm_rows_kernel<<<n_rows, 256, 0, psk::as_stream(stream)>>>(
      h, d, reinterpret_cast<const __nv_bfloat16* const*>(gamma), row_mod, eps,
      reinterpret_cast<__nv_bfloat16*>(out));
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
  rope_append_kernel<<<b->n_rows, 64, 0, psk::as_stream(stream)>>>(
      *b, qkv, n_q_heads, rope, layer, kv, reinterpret_cast<__nv_bfloat16*>(q_rot));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_decode_attn_workspace(const psk_decode_batch* b, int32_t n_kv_heads, int32_t head_dim,
                              int32_t shared_splits, int32_t priv_splits, int64_t* bytes) {
  PSK_CHECK_ARG(b && bytes && head_dim == HD, "psk_decode_attn_workspace: bad args");
  int ns, nt, g;
  attn_items(b, n_kv_heads, shared_splits, priv_splits, &ns, &nt, &g);
  *bytes = (int64_t)nt * AT_GMAX * (HD + 2) * 4;
  return PSK_OK;
}

int psk_decode_attn(const psk_decode_batch* b, const void* q_rot, int32_t n_q_heads, int32_t layer,
                    psk_kv_layout kv, int32_t shared_splits, int32_t priv_splits, void* workspace,
                    void* out, void* stream) {
  PSK_CHECK_ARG(b && q_rot && workspace && out && kv.head_dim == HD && kv.page_tokens == PT &&
                    shared_splits >= 1 && priv_splits >= 1 && n_q_heads % kv.n_kv_heads == 0,
                "psk_decode_attn: bad args");
  const int grp = n_q_heads / kv.n_kv_heads;
  PSK_CHECK_ARG(grp * b->max_rows_per_sess <= AT_GMAX,
                "psk_decode_attn: %d query rows per KV head exceed %d", grp * b->max_rows_per_sess,
                AT_GMAX);
  if (b->n_rows == 0) return PSK_OK;
  AttnParams p;
  p.b = *b;
  p.kv = kv;
  p.q = reinterpret_cast<const __nv_bfloat16*>(q_rot);
  p.nq = n_q_heads;
  p.grp = grp;
  p.layer = layer;
  p.ns_shared = shared_splits;
  p.ns_priv = priv_splits;
  int nt, g;
  attn_items(b, kv.n_kv_heads, shared_splits, priv_splits, &p.n_shared_items, &nt, &g);
  p.gstride = AT_GMAX;
  float* ws = reinterpret_cast<float*>(workspace);
  p.pm = ws;
  p.pl = ws + (int64_t)nt * AT_GMAX;
  p.po = ws + (int64_t)nt * AT_GMAX * 2;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  cudaStream_t s = psk::as_stream(stream);
  static bool attr = false;
  if (!attr) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(decode_attn_partial_kernel,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, AT_SMEM));
    attr = true;
  }
  decode_attn_partial_kernel<<<nt, AT_THREADS, AT_SMEM, s>>>(p);
  PSK_LAUNCH_CHECK();
  decode_attn_merge_kernel<<<dim3(b->n_rows, n_q_heads), HD, 0, s>>>(
      p, reinterpret_cast<__nv_bfloat16*>(out));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_argmax_advance(const psk_decode_batch* b, const float* logits, int32_t vocab,
                       int32_t* out_tokens, int32_t max_new, void* stream) {
  PSK_CHECK_ARG(b && logits && vocab > 0, "psk_argmax_advance: bad args");
  if (b->n_rows == 0) return PSK_OK;
  argmax_advance_kernel<<<b->n_rows, 1024, 0, psk::as_stream(stream)>>>(*b, logits, vocab,
                                                                        out_tokens, max_new);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // extern "C"
