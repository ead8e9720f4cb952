// K3 — causal prefill attention over the paged KV cache, plus the token
// embedding gather of the prefill module.
//
// Reference: softmax(QK^T/sqrt(hd) + causal mask) V per layer
// (frontend/src/model.ts:288-293 mask, :312-315 attention), where new
// positions [pos0, pos0+T) attend to every cached position and causally to
// themselves (a partial prefill after a prefix hit starts at the matched,
// block-aligned pos0: kvstore.py:123-138, cluster.py:322-337).
//
// One CTA = (kv head, block of query positions); its 8 warps are
// (q head of the GQA group) x (16-position sub-block), so each 4 KiB K / V
// page tile is loaded once into XOR-swizzled shared memory (cp.async ring)
// and consumed by every q head of the group. Heavy (late) query blocks are
// scheduled first. Tensor math is mma.sync m16n8k16 (bf16 -> fp32).
#include "common.cuh"
#include "mma.cuh"
#include "tma.cuh"
#include "umma.cuh"

#include <math.h>
#include <stdlib.h>

namespace psk {
namespace pre {

constexpr int HD = 128, PT = 16;
constexpr int WARPS = 8, THREADS = WARPS * 32;
constexpr int RP = 4, NST = 3;
constexpr int TILE = PT * HD * 2;
constexpr int STAGE = RP * 2 * TILE;
constexpr int SMEM = NST * STAGE;  // 96 KiB

__global__ void embed_tokens_kernel(const int64_t* __restrict__ tokens,
                                    const __nv_bfloat16* __restrict__ table, int d,
                                    float* __restrict__ h) {
  const int t = blockIdx.x;
  const __nv_bfloat16* row = table + (int64_t)tokens[t] * d;
  for (int i = threadIdx.x * 8; i < d; i += blockDim.x * 8) {
    float f[8];
    bf16x8_to_f32(*reinterpret_cast<const uint4*>(row + i), f);
    float4* o = reinterpret_cast<float4*>(h + (int64_t)t * d + i);
    o[0] = make_float4(f[0], f[1], f[2], f[3]);
    o[1] = make_float4(f[4], f[5], f[6], f[7]);
  }
}

struct Params {
  const __nv_bfloat16* q;  // [T][nq][HD]
  __nv_bfloat16* out;      // [T][nq*HD]
  psk_kv_layout kv;
  const int32_t* pages;
  int T, pos0, nq, grp, layer;
  int qb;        // query positions per CTA
  int n_qblocks;
  float scale_log2;
};

__device__ __forceinline__ const __nv_bfloat16* tile_ptr(const psk_kv_layout& kv, int page, int layer,
                                                         int kvsel, int head) {
  return reinterpret_cast<const __nv_bfloat16*>(kv.base) + (int64_t)page * kv.page_elems +
         (((int64_t)layer * 2 + kvsel) * kv.n_kv_heads + head) * kv.page_tokens * kv.head_dim;
}

__global__ void __launch_bounds__(THREADS, 2) prefill_attn_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  const int h = blockIdx.x % nkv;
  const int qblk = p.n_qblocks - 1 - (int)(blockIdx.x / nkv);  // heavy blocks first
  const int t0 = qblk * p.qb;                                  // first query (token index)
  const int qh = h * p.grp + warp % p.grp;
  const int sub = warp / p.grp;
  const int wt0 = t0 + sub * 16;                               // this warp's 16 queries
  const bool active = wt0 < p.T;
  const int kv_end = p.pos0 + min(t0 + p.qb, p.T);             // keys [0, kv_end)
  const int n_pages = (kv_end + PT - 1) / PT;
  const int w_last_pos = p.pos0 + min(wt0 + 15, p.T - 1);      // last query position of the warp

  uint32_t qa[8][4];
  {
    const int ta = wt0 + (lane >> 2), tb = ta + 8;
    const int t2 = (lane & 3) * 2;
    const __nv_bfloat16* qA = (active && ta < p.T) ? p.q + ((int64_t)ta * p.nq + qh) * HD : nullptr;
    const __nv_bfloat16* qB = (active && tb < p.T) ? p.q + ((int64_t)tb * p.nq + qh) * HD : nullptr;
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      const int c0 = ks * 16 + t2, c1 = c0 + 8;
      qa[ks][0] = qA ? *reinterpret_cast<const uint32_t*>(qA + c0) : 0u;
      qa[ks][1] = qB ? *reinterpret_cast<const uint32_t*>(qB + c0) : 0u;
      qa[ks][2] = qA ? *reinterpret_cast<const uint32_t*>(qA + c1) : 0u;
      qa[ks][3] = qB ? *reinterpret_cast<const uint32_t*>(qB + c1) : 0u;
    }
  }
  const int posA = p.pos0 + wt0 + (lane >> 2), posB = posA + 8;

  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const int rounds = (n_pages + RP - 1) / RP;
  const uint32_t sbase = smem_u32(smem);
  auto issue = [&](int rd) {
    if (rd < rounds) {
      const uint32_t st = sbase + (rd % NST) * STAGE;
      for (int e = threadIdx.x; e < RP * 2 * 256; e += THREADS) {
        const int ps = e >> 9, kvsel = (e >> 8) & 1, ce = e & 255;
        const int pg = rd * RP + ps;
        if (pg < n_pages) {
          const __nv_bfloat16* src = tile_ptr(p.kv, p.pages[pg], p.layer, kvsel, h);
          const int tr = ce >> 4, c = ce & 15;
          cp_async16(st + (ps * 2 + kvsel) * TILE + swz256(tr, c), src + tr * HD + c * 8);
        }
      }
    }
    cp_async_commit();
  };
#pragma unroll
  for (int s = 0; s < NST - 1; ++s) issue(s);

  for (int rd = 0; rd < rounds; ++rd) {
    cp_async_wait<NST - 2>();
    __syncthreads();
    issue(rd + NST - 1);
    if (!active) continue;
    const uint32_t st = sbase + (rd % NST) * STAGE;
#pragma unroll 1
    for (int ps = 0; ps < RP; ++ps) {
      const int pg = rd * RP + ps;
      if (pg >= n_pages) break;
      const int key0 = pg * PT;
      if (key0 > w_last_pos) break;  // fully in the causal future of this warp
      const uint32_t kt = st + (ps * 2) * TILE, vt = kt + TILE;
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
      const int cb = (lane & 3) * 2;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = key0 + nt * 8 + cb + (e & 1);
          const int qpos = (e < 2) ? posA : posB;
          s[nt][e] = (key <= qpos && key < kv_end) ? s[nt][e] * p.scale_log2 : -INFINITY;
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
  cp_async_wait<0>();
  if (!active) return;
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float i0 = l0 > 0.f ? 1.f / l0 : 0.f, i1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int ta = wt0 + (lane >> 2), tb = ta + 8;
  const int cb = (lane & 3) * 2;
#pragma unroll
  for (int nt = 0; nt < 16; ++nt) {
    if (ta < p.T)
      *reinterpret_cast<__nv_bfloat162*>(p.out + ((int64_t)ta * p.nq + qh) * HD + nt * 8 + cb) =
          __floats2bfloat162_rn(o[nt][0] * i0, o[nt][1] * i0);
    if (tb < p.T)
      *reinterpret_cast<__nv_bfloat162*>(p.out + ((int64_t)tb * p.nq + qh) * HD + nt * 8 + cb) =
          __floats2bfloat162_rn(o[nt][2] * i1, o[nt][3] * i1);
  }
}

// ------------------------------------------------------ tcgen05 variant ----
// Causal prefill attention on the 5th-gen tensor cores. One CTA = (kv head,
// block of 128/grp query positions x grp q heads = 128 query rows). Per
// 8-page chunk (128 keys): S = Q.K^T and D = P.V are UMMAs (M=128, N=128)
// with TMEM accumulators; a TMA producer warp streams K/V chunks (K boxes
// laid out at a uniform 128 B row stride across the chunk's pages, V as an
// MN-major operand); 4 softmax warps own one query row each (thread = TMEM
// lane), apply the causal mask, write bf16 P in the UMMA K-major SW128 layout
// and keep O in registers with the online-softmax rescale.
namespace tc {

constexpr int CP = 8, NSTG = 2;
constexpr int KREG = CP * TILE, VREG = CP * TILE, STG = KREG + VREG;  // 32 + 32 KiB
constexpr int OFF_Q = NSTG * STG;
constexpr int OFF_P = OFF_Q + 32768;
constexpr int OFF_BAR = OFF_P + 32768;
constexpr int MAXPG = 2560;  // page table staged in smem (40k tokens)
constexpr int OFF_PG = OFF_BAR + 256;
constexpr int SMEM = OFF_PG + MAXPG * 4 + 1024;
constexpr int THREADS_TC = 192;
constexpr int TMEM_COLS = 256;

struct TcParams {
  const __nv_bfloat16* q;
  __nv_bfloat16* out;
  psk_kv_layout kv;
  const int32_t* pages;
  int T, pos0, nq, grp, layer, qb, n_qblocks;
  float scale_log2;
  // batched (varlen) prefill: per work item 8 ints {token offset of the
  // sequence in q/out, T, pos0, offset of its page table in `pages`, q-block,
  // 0, 0, 0}; nullptr = one sequence (T, pos0, pages), q-blocks heavy first
  const int32_t* items;
};

__global__ void __launch_bounds__(THREADS_TC, 1)
    prefill_attn_tc(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ TcParams p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t *full = bars, *empty = bars + 2, *s_full = bars + 4, *s_empty = bars + 5, *p_full = bars + 6,
           *d_full = bars + 7, *d_empty = bars + 8;
  int* s_pg = reinterpret_cast<int*>(smem + OFF_PG);
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  const int h = blockIdx.x % nkv;
  const int qblk = p.n_qblocks - 1 - (int)(blockIdx.x / nkv);  // heavy blocks first
  const int t0 = qblk * p.qb;
  const int kv_end = p.pos0 + min(t0 + p.qb, p.T);
  const int n_pages = (kv_end + PT - 1) / PT;
  const int nch = (n_pages + CP - 1) / CP;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], 1);
    }
    tma::mbar_init(s_full, 1);
    tma::mbar_init(s_empty, 128);
    tma::mbar_init(p_full, 128);
    tma::mbar_init(d_full, 1);
    tma::mbar_init(d_empty, 128);
    tma::fence_mbar_init();
    tma::prefetch_map(&kvmap);
  }
  if (warp == 1) umma::tmem_alloc(&s_tmem, TMEM_COLS);
  for (int j = threadIdx.x; j < n_pages && j < MAXPG; j += THREADS_TC) s_pg[j] = p.pages[j];
  const uint32_t sq = smem_u32(smem + OFF_Q), sp = smem_u32(smem + OFF_P);
  for (int e = threadIdx.x; e < 128 * 16; e += THREADS_TC) {
    const int g = e >> 4, c = e & 15;
    const int t = t0 + g / p.grp;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t < p.T) {
      const int qh = h * p.grp + g % p.grp;
      v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)t * p.nq + qh) * HD + c * 8);
    }
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sq + umma::kmajor_off(g, c, 16384)), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w));
  }
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = s_tmem;

  if (warp == 0) {
    if (lane == 0) {
      for (int c = 0; c < nch; ++c) {
        const int st = c % NSTG;
        tma::mbar_wait(&empty[st], ((c / NSTG) & 1) ^ 1);
        tma::mbar_expect_tx(&full[st], STG);
        unsigned char* kr = smem + st * STG;
        unsigned char* vr = kr + KREG;
        for (int pp = 0; pp < CP; ++pp) {
          const int j = c * CP + pp;
          const int jj = j < n_pages ? j : c * CP;  // past the end: any valid page, masked
          const int page = jj < MAXPG ? s_pg[jj] : p.pages[jj];
          const int row_k = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv + h) * PT);
          const int row_v = row_k + nkv * PT;
          tma::load_2d(&kvmap, &full[st], kr + pp * 2048, 0, row_k);
          tma::load_2d(&kvmap, &full[st], kr + CP * 2048 + pp * 2048, 64, row_k);
          tma::load_2d(&kvmap, &full[st], vr + pp * TILE, 0, row_v);
          tma::load_2d(&kvmap, &full[st], vr + pp * TILE + 2048, 64, row_v);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t ID_QK = umma::idesc_bf16(128, 128, false), ID_PV = umma::idesc_bf16(128, 128, true);
      for (int c = 0; c < nch; ++c) {
        const int st = c % NSTG;
        const uint32_t kr = smem_u32(smem + st * STG), vr = kr + KREG;
        tma::mbar_wait(&full[st], (c / NSTG) & 1);
        tma::mbar_wait(s_empty, (c & 1) ^ 1);
        umma::fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma::mma(tmem, umma::desc_k_sw128(sq + (kk >> 2) * 16384) + 2 * (kk & 3),
                    umma::desc_k_sw128(kr + (kk >> 2) * (CP * 2048)) + 2 * (kk & 3), ID_QK, kk > 0);
        umma::commit(s_full);
        tma::mbar_wait(p_full, c & 1);
        tma::mbar_wait(d_empty, (c & 1) ^ 1);
        umma::fence_after();
#pragma unroll
        for (int pp = 0; pp < CP; ++pp)
          umma::mma(tmem + 128, umma::desc_k_sw128(sp + (pp >> 2) * 16384) + 2 * (pp & 3),
                    umma::desc_mn_sw128(vr + pp * TILE, 2048), ID_PV, pp > 0);
        umma::commit(d_full);
        umma::commit(&empty[st]);
      }
    }
  } else {
    const int q4 = warp & 3;
    const int g = q4 * 32 + lane;
    const uint32_t tS = tmem + ((uint32_t)(q4 * 32) << 16), tD = tS + 128;
    const int t = t0 + g / p.grp;
    const int qpos = p.pos0 + t;  // keys [0, qpos] are visible
    float O[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) O[i] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int c = 0; c < nch; ++c) {
      const int key0 = c * CP * PT;
      tma::mbar_wait(s_full, c & 1);
      umma::fence_after();
      float v[16];
      float mx = -INFINITY;
#pragma unroll
      for (int gi = 0; gi < 8; ++gi) {
        umma::ld16(tS + gi * 16, v);
#pragma unroll
        for (int e = 0; e < 16; ++e)
          if (key0 + gi * 16 + e <= qpos) mx = fmaxf(mx, v[e] * p.scale_log2);
      }
      const float mn = fmaxf(m, mx);
      const float base = mn == -INFINITY ? 0.f : mn;
      const float alpha = exp2f(m - base);
      float ladd = 0.f;
#pragma unroll
      for (int gi = 0; gi < 8; ++gi) {
        umma::ld16(tS + gi * 16, v);
        uint32_t pk[8];
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          const int key = key0 + gi * 16 + e;
          const float p0 = key <= qpos ? exp2f(v[e] * p.scale_log2 - base) : 0.f;
          const float p1 = key + 1 <= qpos ? exp2f(v[e + 1] * p.scale_log2 - base) : 0.f;
          ladd += p0 + p1;
          pk[e >> 1] = pack_bf16(p0, p1);
        }
#pragma unroll
        for (int cc = 0; cc < 2; ++cc)
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sp + umma::kmajor_off(g, gi * 2 + cc, 16384)),
                       "r"(pk[4 * cc]), "r"(pk[4 * cc + 1]), "r"(pk[4 * cc + 2]), "r"(pk[4 * cc + 3]));
      }
      umma::fence_before();
      tma::mbar_arrive(s_empty);
      umma::fence_proxy_async();
      tma::mbar_arrive(p_full);
      l = l * alpha + ladd;
      tma::mbar_wait(d_full, c & 1);
      umma::fence_after();
#pragma unroll
      for (int gi = 0; gi < 8; ++gi) {
        umma::ld16(tD + gi * 16, v);
#pragma unroll
        for (int e = 0; e < 16; ++e) O[gi * 16 + e] = O[gi * 16 + e] * alpha + v[e];
      }
      umma::fence_before();
      tma::mbar_arrive(d_empty);
      m = mn;
    }
    if (t < p.T) {
      const float inv = l > 0.f ? 1.f / l : 0.f;
      const int qh = h * p.grp + g % p.grp;
      uint4* dst = reinterpret_cast<uint4*>(p.out + ((int64_t)t * p.nq + qh) * HD);
#pragma unroll
      for (int i = 0; i < HD / 8; ++i) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = O[8 * i + e] * inv;
        dst[i] = f32_to_bf16x8(f);
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 1) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, TMEM_COLS);
  }
}

}  // namespace tc

// ------------------------------------------------------ ping-pong tcgen05 ---
// One CTA = (kv head, 256 query rows = two 128-row tiles of (position, q
// head of the GQA group)); both tiles consume every 64-key K/V chunk.
//   warp 0      TMA producer: K and V of 4 pages per chunk, 3-stage ring
//   warp 1      MMA issuer (+ TMEM owner): S_t = Q_t K^T (M128 N64), then
//               O_t += P_t V (M128 N128 K16 per page); issue order
//               PV0(c) S0(c+1) PV1(c) S1(c+1) so one tile's softmax runs
//               while the tensor core works on the other tile
//   softmax     SPLIT = 2 (default): warps 2-9 tile 0, 10-17 tile 1, two
//               threads per query row (TMEM lane), 32 keys each, their
//               partial row maxima swapped through shared memory per chunk;
//               SPLIT = 1 (PSK_PREFILL_SPLIT=1): warps 2-5 / 6-9, a thread per
//               row. One pass over S from TMEM, exp2 with a lazily updated
//               base max (O in TMEM is rescaled only when the row max grows
//               by > 2^8; the final 1/l makes it exact), P (bf16) -> TMEM,
//               double-buffered per tile, so softmax(c+1) never waits for
//               PV(c); the PV MMA takes P as its A operand from tensor memory
// TMEM columns: S0 [0,64) S1 [64,128) O0 [128,256) O1 [256,384)
//               P[tile][buffer] [384 + 32 (2 tile + buffer), +32) (bf16 pairs).
// The producer and MMA warps run warp-converged (all 32 lanes, warp-uniform
// operands, one elected lane issues): from an if (lane == 0) branch the
// compiler wraps every TMA / MMA in an R2UR.BROADCAST waterfall loop.
#ifndef PP_EMU
// K3 softmax: exponentials per 8 computed on the FMA pipe (exp2_fma). Off:
// alternating A/B at 4k (tools/ab_prefill.sh) measured 188 us/layer with 0,
// 202 with 3, 217 with 2, 238 with 4 -- MUFU is not this kernel's limiter.
#define PP_EMU 0
#endif

namespace pp {

constexpr int KC = 64;                   // keys per chunk
constexpr int CPG = KC / PT;             // pages per chunk
constexpr int NSTG = 3;
constexpr int KBYTES = CPG * TILE;       // 16 KiB: [dims 0-63 box x 4 pages][dims 64-127 box x 4 pages]
constexpr int STG = 2 * KBYTES;          // + V 16 KiB: [page][box0 | box1]
constexpr int QBYTES = 128 * HD * 2;     // 32 KiB per tile: [2 boxes][128 rows][128 B]
constexpr int OFF_Q = NSTG * STG;
constexpr int OFF_XCH = OFF_Q + 2 * QBYTES;  // SPLIT = 2: row max / sum exchange [tile][half][parity][128] fp32
constexpr int OFF_BAR = OFF_XCH + 4096;
constexpr int MAXPG = 2560;
constexpr int OFF_PG = OFF_BAR + 256;
constexpr int SMEM = OFF_PG + MAXPG * 4 + 1024;
constexpr float RESCALE_LOG2 = 8.f;      // lazy-rescale threshold (log2 units)
constexpr uint32_t T_P = 384;            // P buffers in TMEM
constexpr int threads_of(int split) { return 64 + 2 * 128 * split; }

// SPLIT softmax threads per query row: 1 (one row per thread, the round-1
// layout) or 2 (each thread takes 32 of a chunk's 64 keys; the pair -- same
// TMEM lane quarter, warps 4 apart -- swaps its partial row maxima through
// shared memory once per chunk, keeps its own partial row sum, and rescales
// / writes its half of the O row). SPLIT = 2 doubles the softmax warps in
// flight (18 warps per CTA) for the same work.
template <int SPLIT>
__global__ void __launch_bounds__(threads_of(SPLIT), 1)
    prefill_attn_pp(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ tc::TcParams p) {
  constexpr int THREADS = threads_of(SPLIT);
  constexpr int NC = KC / SPLIT;  // keys per softmax thread per chunk
  constexpr int OC = HD / SPLIT;  // O columns per softmax thread
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  // pv_done[2 t + b]: PV_t of the chunks c with c % 2 == b (P buffer b)
  uint64_t *full = bars, *empty = bars + NSTG, *s_full = bars + 2 * NSTG, *p_full = s_full + 2,
           *pv_done = p_full + 2, *s_free = pv_done + 4;
  int* s_pg = reinterpret_cast<int*>(smem + OFF_PG);
  float* xch = reinterpret_cast<float*>(smem + OFF_XCH);
  __shared__ uint32_t s_tmem;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  const int h = blockIdx.x % nkv;
  int qblk, T = p.T, pos0 = p.pos0;
  const int32_t* pages = p.pages;
  const __nv_bfloat16* qsrc = p.q;
  __nv_bfloat16* odst = p.out;
  if (p.items != nullptr) {  // batched prefill: this CTA's (sequence, q-block)
    const int4 it = reinterpret_cast<const int4*>(p.items)[2 * (blockIdx.x / nkv)];
    const int qb_ = reinterpret_cast<const int4*>(p.items)[2 * (blockIdx.x / nkv) + 1].x;
    qsrc += (int64_t)it.x * p.nq * HD;
    odst += (int64_t)it.x * p.nq * HD;
    T = it.y;
    pos0 = it.z;
    pages += it.w;
    qblk = qb_;
  } else {
    qblk = p.n_qblocks - 1 - (int)(blockIdx.x / nkv);  // heavy blocks first
  }
  const int t0 = qblk * p.qb;  // p.qb = 256 / grp positions
  const int kv_end = pos0 + min(t0 + p.qb, T);
  const int n_pages = (kv_end + PT - 1) / PT;
  const int nch = (kv_end + KC - 1) / KC;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTG; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], 1);
    }
    for (int t = 0; t < 2; ++t) {
      tma::mbar_init(&s_full[t], 1);
      tma::mbar_init(&s_free[t], 128 * SPLIT);
      tma::mbar_init(&p_full[t], 128 * SPLIT);
      tma::mbar_init(&pv_done[2 * t], 1);
      tma::mbar_init(&pv_done[2 * t + 1], 1);
    }
    tma::fence_mbar_init();
    tma::prefetch_map(&kvmap);
  }
  if (warp == 1) umma::tmem_alloc(&s_tmem, 512);
  for (int j = threadIdx.x; j < n_pages && j < MAXPG; j += THREADS) s_pg[j] = pages[j];
  const uint32_t sq = smem_u32(smem + OFF_Q);
  // PDL: the page table and items are host-written before the forward; q and
  // the layer's K/V come from the QKV GEMM just before this kernel
  psk::pdl_wait();
  // Q rows -> shared memory (K-major, 128B swizzle), row r = (position, head)
  for (int e = threadIdx.x; e < 256 * 16; e += THREADS) {
    const int r = e >> 4, c = e & 15;
    const int t = t0 + r / p.grp;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t < T) {
      const int qh = h * p.grp + r % p.grp;
      v = *reinterpret_cast<const uint4*>(qsrc + ((int64_t)t * p.nq + qh) * HD + c * 8);
    }
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(sq + (r >> 7) * QBYTES +
                                                               umma::kmajor_off(r & 127, c, 16384)),
                 "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
  }
  umma::fence_proxy_async();
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  const uint32_t tmem = s_tmem;
  psk::pdl_trigger();

  if (warp == 0) {
    for (int c = 0; c < nch; ++c) {
      const int st = c % NSTG;
      tma::mbar_wait(&empty[st], ((c / NSTG) & 1) ^ 1);
      tma::mbar_expect_tx_e(&full[st], STG);
      unsigned char* kr = smem + st * STG;
      unsigned char* vr = kr + KBYTES;
#pragma unroll
      for (int pp = 0; pp < CPG; ++pp) {
        const int j = c * CPG + pp;
        const int jj = j < n_pages ? j : c * CPG;  // past the end: any valid page, masked
        const int page = jj < MAXPG ? s_pg[jj] : pages[jj];
        const int row_k = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv + h) * PT);
        const int row_v = row_k + nkv * PT;
        tma::load_2d_e(&kvmap, &full[st], kr + pp * 2048, 0, row_k);
        tma::load_2d_e(&kvmap, &full[st], kr + CPG * 2048 + pp * 2048, 64, row_k);
        tma::load_2d_e(&kvmap, &full[st], vr + pp * TILE, 0, row_v);
        tma::load_2d_e(&kvmap, &full[st], vr + pp * TILE + 2048, 64, row_v);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t ID_S = umma::idesc_bf16(128, KC, false), ID_PV = umma::idesc_bf16(128, HD, true);
    auto issue_s = [&](int t, int c) {
      const uint32_t kr = smem_u32(smem + (c % NSTG) * STG);
      const uint32_t qt = sq + t * QBYTES;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        umma::mma_e(tmem + t * KC, umma::desc_k_sw128(qt + (kk >> 2) * 16384) + 2 * (kk & 3),
                    umma::desc_k_sw128(kr + (kk >> 2) * (CPG * 2048)) + 2 * (kk & 3), ID_S, kk > 0);
      umma::commit_e(&s_full[t]);
    };
    auto issue_pv = [&](int t, int c) {
      const uint32_t vr = smem_u32(smem + (c % NSTG) * STG) + KBYTES;
      const uint32_t pt = tmem + T_P + (2 * t + (c & 1)) * (KC / 2);
#pragma unroll
      for (int pp = 0; pp < CPG; ++pp)
        umma::mma_ts_e(tmem + 128 + t * HD, pt + pp * 8, umma::desc_mn_sw128(vr + pp * TILE, 2048), ID_PV,
                       (c > 0 || pp > 0) ? 1u : 0u);
      umma::commit_e(&pv_done[2 * t + (c & 1)]);
    };
    tma::mbar_wait(&full[0], 0);
    umma::fence_after();
    issue_s(0, 0);
    issue_s(1, 0);
    for (int c = 0; c < nch; ++c) {
      const bool more = c + 1 < nch;
      if (more) tma::mbar_wait(&full[(c + 1) % NSTG], ((c + 1) / NSTG) & 1);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        // S_t(c+1) as soon as softmax(c) holds S_t(c) in registers (it runs
        // under that softmax), PV_t(c) once P_t(c) is written
        if (more) {
          tma::mbar_wait(&s_free[t], c & 1);
          umma::fence_after();
          issue_s(t, c + 1);
        }
        tma::mbar_wait(&p_full[t], c & 1);  // P_t(c) written
        umma::fence_after();
        issue_pv(t, c);
      }
      umma::commit_e(&empty[c % NSTG]);  // K/V stage free once both PVs completed
    }
  } else {
    const int sw = warp - 2;
    const int t = sw >> (SPLIT == 2 ? 3 : 2);            // tile
    const int hf = SPLIT == 2 ? (sw >> 2) & 1 : 0;       // half of the chunk's keys / of the O row
    const int lq = (warp & 3) * 32;                      // TMEM lane quarter of this warp
    const int g = lq + lane;                             // row in the tile
    const int r = t * 128 + g;                           // row in the CTA
    const int bar_id = 1 + t * 4 + (warp & 3);           // SPLIT = 2: the pair's named barrier
    const uint32_t tS = tmem + ((uint32_t)lq << 16) + t * KC + hf * NC;
    const uint32_t tO = tmem + ((uint32_t)lq << 16) + 128 + t * HD + hf * OC;
    const uint32_t tP = tmem + ((uint32_t)lq << 16) + T_P + hf * (NC / 2);
    const int qpos = pos0 + t0 + r / p.grp;  // keys [0, qpos] visible
    float m_used = -INFINITY, l = 0.f;
    for (int c = 0; c < nch; ++c) {
      const int key0 = c * KC + hf * NC;
      tma::mbar_wait(&s_full[t], c & 1);
      umma::fence_after();
      uint32_t sr[NC];
#pragma unroll
      for (int k = 0; k < NC / 32; ++k) umma::ld32_async(tS + 32 * k, sr + 32 * k);
      umma::wait_ld();
      umma::fence_before();
      tma::mbar_arrive(&s_free[t]);  // S_t may be overwritten by S_t(c+1)
      // causal mask only on the chunks that cross the warp's diagonal
      if (!__all_sync(0xffffffffu, key0 + NC - 1 <= qpos)) {
#pragma unroll
        for (int e = 0; e < NC; ++e)
          if (key0 + e > qpos) sr[e] = __float_as_uint(-INFINITY);
      }
      // tree max of the raw scores (no serial chain), then into log2 units
      float tm[NC / 2];
#pragma unroll
      for (int k = 0; k < NC / 2; ++k) tm[k] = fmaxf(__uint_as_float(sr[2 * k]), __uint_as_float(sr[2 * k + 1]));
#pragma unroll
      for (int w = NC / 4; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) tm[k] = fmaxf(tm[k], tm[k + w]);
      float rmax = tm[0];
      if (SPLIT == 2) {  // the row's other half (double-buffered by chunk parity)
        xch[((t * 2 + hf) * 2 + (c & 1)) * 128 + g] = rmax;
        named_barrier_sync(bar_id, 64);
        rmax = fmaxf(rmax, xch[((t * 2 + (hf ^ 1)) * 2 + (c & 1)) * 128 + g]);
      }
      const float mx = rmax * p.scale_log2;
      // PV_t(c-2) before P buffer c % 2 is overwritten; PV_t(c-1) only
      // before a rescale of O_t
      if (c > 1) tma::mbar_wait(&pv_done[2 * t + (c & 1)], ((c >> 1) - 1) & 1);
      const bool grow = mx > m_used + RESCALE_LOG2 || (m_used == -INFINITY && mx > -INFINITY);
      if (__any_sync(0xffffffffu, grow && c > 0)) {
        tma::mbar_wait(&pv_done[2 * t + ((c - 1) & 1)], ((c - 1) >> 1) & 1);
        umma::fence_after();
        const float alpha = grow ? exp2f(m_used - mx) : 1.f;
#pragma unroll 1
        for (int q = 0; q < OC / 32; ++q) {
          uint32_t o[32];
          umma::ld32_async(tO + q * 32, o);
          umma::wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
          umma::st32(tO + q * 32, o);
        }
        umma::wait_st();
        l *= alpha;
      }
      if (grow) m_used = mx;
      const float base = m_used == -INFINITY ? 0.f : m_used;
      float ls[NC / 8];
      uint32_t pk[NC / 2];
#pragma unroll
      for (int q = 0; q < NC / 8; ++q) {
        float pf[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {  // p = 2^(s * scale - m); masked: 2^-inf = 0
          const float x = fmaf(__uint_as_float(sr[8 * q + i]), p.scale_log2, -base);
          // PP_EMU of every 8 exponentials on the FMA pipe, the rest on MUFU
          pf[i] = i >= 8 - PP_EMU ? exp2_fma(x) : fast_exp2(x);
        }
        ls[q] = ((pf[0] + pf[1]) + (pf[2] + pf[3])) + ((pf[4] + pf[5]) + (pf[6] + pf[7]));
        const uint4 v = f32_to_bf16x8(pf);
        pk[4 * q] = v.x;
        pk[4 * q + 1] = v.y;
        pk[4 * q + 2] = v.z;
        pk[4 * q + 3] = v.w;
      }
#pragma unroll
      for (int w = NC / 16; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) ls[k] += ls[k + w];
      l += ls[0];
      if (SPLIT == 2)
        umma::st16(tP + (2 * t + (c & 1)) * (KC / 2), pk);
      else
        umma::st32(tP + (2 * t + (c & 1)) * (KC / 2), pk);
      umma::wait_st();
      umma::fence_before();
      tma::mbar_arrive(&p_full[t]);
    }
    if (SPLIT == 2) {  // the row sum: this half's + the other's
      named_barrier_sync(bar_id, 64);  // the last chunk's max reads are done
      xch[(t * 2 + hf) * 2 * 128 + g] = l;
      named_barrier_sync(bar_id, 64);
      l += xch[(t * 2 + (hf ^ 1)) * 2 * 128 + g];
    }
    // epilogue: this thread's OC columns of O_t / l -> bf16 row of the output
    tma::mbar_wait(&pv_done[2 * t + ((nch - 1) & 1)], ((nch - 1) >> 1) & 1);
    umma::fence_after();
    const int tpos = t0 + r / p.grp;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* dst = odst + ((int64_t)tpos * p.nq + h * p.grp + r % p.grp) * HD + hf * OC;
#pragma unroll 1
    for (int q = 0; q < OC / 32; ++q) {
      uint32_t o[32];
      umma::ld32_async(tO + q * 32, o);
      umma::wait_ld();
      if (tpos < T) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          float f[8];
#pragma unroll
          for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(o[8 * i + e]) * inv;
          reinterpret_cast<uint4*>(dst + q * 32)[i] = f32_to_bf16x8(f);
        }
      }
    }
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 1) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, 512);
  }
}

typedef void (*KernelFn)(const CUtensorMap, const tc::TcParams);
struct Variant {
  KernelFn fn;
  int threads;
};

// The K3 variant in use (PSK_PREFILL_SPLIT=1: one softmax thread per row),
// its shared-memory attribute set once.
static Variant kernel() {
  static Variant v{nullptr, 0};
  if (!v.fn) {
    const bool one = getenv("PSK_PREFILL_SPLIT") && getenv("PSK_PREFILL_SPLIT")[0] == '1';
    const Variant c = one ? Variant{prefill_attn_pp<1>, threads_of(1)} : Variant{prefill_attn_pp<2>, threads_of(2)};
    if (cudaFuncSetAttribute(c.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM) != cudaSuccess) return c;
    v = c;
  }
  return v;
}

}  // namespace pp

}  // namespace pre
}  // namespace psk

extern "C" {

int psk_embed_tokens(const int64_t* tokens, int32_t T, const void* table, int32_t d, float* h,
                     void* stream) {
  PSK_CHECK_ARG(tokens && table && h && d % 8 == 0 && T >= 0, "psk_embed_tokens: bad args");
  if (T == 0) return PSK_OK;
  psk::pre::embed_tokens_kernel<<<T, 128, 0, psk::as_stream(stream)>>>(
      tokens, reinterpret_cast<const __nv_bfloat16*>(table), d, h);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_prefill_attn(const void* q_rot, int32_t T, int32_t pos0, int32_t n_q_heads, psk_kv_layout kv,
                     int32_t layer, const int32_t* page_table, void* out, void* stream) {
  using namespace psk::pre;
  PSK_CHECK_ARG(q_rot && page_table && out && kv.head_dim == HD && kv.page_tokens == PT &&
                    n_q_heads % kv.n_kv_heads == 0,
                "psk_prefill_attn: bad args");
  const int grp = n_q_heads / kv.n_kv_heads;
  PSK_CHECK_ARG(grp >= 1 && grp <= WARPS && WARPS % grp == 0, "psk_prefill_attn: GQA group %d", grp);
  if (T == 0) return PSK_OK;
  Params p;
  p.q = reinterpret_cast<const __nv_bfloat16*>(q_rot);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.kv = kv;
  p.pages = page_table;
  p.T = T;
  p.pos0 = pos0;
  p.nq = n_q_heads;
  p.grp = grp;
  p.layer = layer;
  p.qb = 16 * (WARPS / grp);
  p.n_qblocks = (T + p.qb - 1) / p.qb;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  static const bool force_hmma = getenv("PSK_PREFILL_HMMA") != nullptr;
  if (!force_hmma && kv.n_pages > 0 && 128 % grp == 0) {
    CUtensorMap map;
    int rc = psk::kv_tensor_map(kv, &map);
    if (rc) return rc;
    tc::TcParams t;
    t.q = p.q;
    t.out = p.out;
    t.kv = kv;
    t.pages = page_table;
    t.T = T;
    t.pos0 = pos0;
    t.nq = n_q_heads;
    t.grp = grp;
    t.layer = layer;
    t.scale_log2 = p.scale_log2;
    t.items = nullptr;
    static const bool tc1 = getenv("PSK_PREFILL_TC1") != nullptr;
    if (!tc1) {
      t.qb = 256 / grp;
      t.n_qblocks = (T + t.qb - 1) / t.qb;
      const pp::Variant v = pp::kernel();
      PSK_CUDA_TRY(psk::launch_pdl(v.fn, dim3(t.n_qblocks * kv.n_kv_heads), dim3(v.threads), (size_t)pp::SMEM,
                                   psk::as_stream(stream), map, t));
      PSK_LAUNCH_CHECK();
      return PSK_OK;
    }
    t.qb = 128 / grp;
    t.n_qblocks = (T + t.qb - 1) / t.qb;
    static bool tc_attr = false;
    if (!tc_attr) {
      PSK_CUDA_TRY(cudaFuncSetAttribute(tc::prefill_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        tc::SMEM));
      tc_attr = true;
    }
    tc::prefill_attn_tc<<<t.n_qblocks * kv.n_kv_heads, tc::THREADS_TC, tc::SMEM, psk::as_stream(stream)>>>(
        map, t);
    PSK_LAUNCH_CHECK();
    return PSK_OK;
  }
  static bool attr = false;
  if (!attr) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(prefill_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM));
    attr = true;
  }
  prefill_attn_kernel<<<p.n_qblocks * kv.n_kv_heads, THREADS, SMEM, psk::as_stream(stream)>>>(p);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_prefill_attn_batch(const void* q_rot, int32_t n_items, const int32_t* items, int32_t n_q_heads,
                           psk_kv_layout kv, int32_t layer, const int32_t* pages, void* out, void* stream) {
  using namespace psk::pre;
  PSK_CHECK_ARG(q_rot && items && pages && out && kv.head_dim == HD && kv.page_tokens == PT && kv.n_pages > 0 &&
                    n_q_heads % kv.n_kv_heads == 0 && n_items >= 0,
                "psk_prefill_attn_batch: bad args");
  const int grp = n_q_heads / kv.n_kv_heads;
  PSK_CHECK_ARG(128 % grp == 0, "psk_prefill_attn_batch: GQA group %d", grp);
  if (n_items == 0) return PSK_OK;
  CUtensorMap map;
  int rc = psk::kv_tensor_map(kv, &map);
  if (rc) return rc;
  tc::TcParams t{};
  t.q = reinterpret_cast<const __nv_bfloat16*>(q_rot);
  t.out = reinterpret_cast<__nv_bfloat16*>(out);
  t.kv = kv;
  t.pages = pages;
  t.nq = n_q_heads;
  t.grp = grp;
  t.layer = layer;
  t.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  t.qb = 256 / grp;
  t.items = items;
  const pp::Variant v = pp::kernel();
  PSK_CUDA_TRY(psk::launch_pdl(v.fn, dim3(n_items * kv.n_kv_heads), dim3(v.threads), (size_t)pp::SMEM,
                               psk::as_stream(stream), map, t));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // extern "C"
