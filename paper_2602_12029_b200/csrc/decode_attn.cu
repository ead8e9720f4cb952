// K6 — shared-prefix paged decode attention (one launch per layer).
//
// Decode modules batched on one session share the base module's prompt KV
// (the PrefillShare cache reuse: frontend/src/evaluate.ts:21-50, one base
// cache consumed by several decoders; the reference re-concatenates and
// re-reads the full past per model and per step, model.ts:307-315). Here one
// thread-block CLUSTER serves one (session, KV head):
//
//   * the page stream is [shared prompt pages | row 0 private pages | row 1
//     private pages | ...]; every page is fetched from HBM exactly once per
//     step by TMA (128B-swizzled 4 KiB K and V tiles) into a 12-stage ring
//     driven by a producer warp, and consumed by ALL query rows of the
//     session (GQA group x co-batched decode modules, <= 64 rows = 4 MMA
//     tiles); private pages mask the rows they do not belong to;
//   * the C CTAs of the cluster split the stream; each CTA folds its warps'
//     online-softmax partials in shared memory, then the cluster reduces the
//     C partials through distributed shared memory (DSMEM) and writes the
//     normalised bf16 output — no global partials, no second kernel.
#include "common.cuh"
#include "mma.cuh"
#include "tma.cuh"

#include <math.h>

namespace psk {
namespace dattn {

constexpr int HD = 128, PT = 16;
constexpr int CW = 8;                 // consumer warps
constexpr int THREADS = (CW + 1) * 32;  // + 1 TMA producer warp
constexpr int NST = 12;               // pipeline stages (1 page each)
constexpr int TILE = PT * HD * 2;     // 4 KiB
constexpr int STAGE = 2 * TILE;       // K + V
constexpr int GMAX = 64;
constexpr int MAXR = 16;              // rows per session
constexpr int OFF_Q = NST * STAGE;                  // 96 KiB
constexpr int OFF_O = OFF_Q + GMAX * 256;           // +16 KiB
constexpr int OFF_M = OFF_O + GMAX * HD * 4;        // +32 KiB
constexpr int OFF_L = OFF_M + GMAX * 4;
constexpr int OFF_BAR = OFF_L + GMAX * 4;
constexpr int SMEM = OFF_BAR + 2 * NST * 8 + 1024;  // + alignment slack

struct Params {
  psk_decode_batch b;
  psk_kv_layout kv;
  const __nv_bfloat16* q;  // [rows][nq][HD]
  __nv_bfloat16* out;      // [rows][nq][HD]
  int nq, grp, layer;
  float scale_log2;
};

struct PageMeta {
  int page, limit, owner;  // owner: -1 shared, else row index within session
};

// SW128 address of (token row, 16-byte chunk c16 in 0..15) in a K/V tile made
// of two [16 x 128 B] TMA boxes (dims 0-63, 64-127).
__device__ __forceinline__ uint32_t tile_addr(uint32_t tile, int tok, int c16) {
  return tile + ((c16 >> 3) << 11) + tok * 128 + (((c16 & 7) ^ (tok & 7)) << 4);
}

template <int C>
__global__ void __launch_bounds__(THREADS, 1)
    decode_attn_kernel(const __grid_constant__ CUtensorMap kvmap, Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* empty = full + NST;
  float* sO = reinterpret_cast<float*>(smem + OFF_O);
  float* sM = reinterpret_cast<float*>(smem + OFF_M);
  float* sL = reinterpret_cast<float*>(smem + OFF_L);
  __shared__ int s_rows[MAXR], s_plen[MAXR], s_pstart[MAXR + 1];
  __shared__ int s_ps, s_ls, s_total;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  const int cl = blockIdx.x / C;
  const int rank = (int)tma::cluster_rank();
  const int sess = cl / nkv, h = cl % nkv;
  const int nr = p.b.sess_nrows[sess];
  const int G = nr * p.grp;
  const int T = (G + 15) / 16;
  const int Tp = T <= 1 ? 1 : (T == 2 ? 2 : 4);
  const int ways = CW / Tp;

  if (threadIdx.x == 0) {
    const int Ls = p.b.sess_len[sess];
    const int Ps = (Ls + PT - 1) / PT;
    s_ls = Ls;
    s_ps = Ps;
    int acc = Ps;
    for (int i = 0; i < nr; ++i) {
      const int r = p.b.sess_rows[(int64_t)sess * p.b.max_rows_per_sess + i];
      const int lp = p.b.priv_len[r] + 1;  // includes the token appended this step
      s_rows[i] = r;
      s_plen[i] = lp;
      s_pstart[i] = acc;
      acc += (lp + PT - 1) / PT;
    }
    s_pstart[nr] = acc;
    s_total = acc;
    for (int s = 0; s < NST; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], T);
    }
    tma::fence_mbar_init();
    tma::prefetch_map(&kvmap);
  }
  // Q tile -> shared (swizzled 256 B rows), zero rows beyond G
  {
    const uint32_t qs = smem_u32(smem + OFF_Q);
    for (int e = threadIdx.x; e < T * 16 * 16; e += THREADS) {
      const int g = e >> 4, c = e & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (g < G) {
        const int r = p.b.sess_rows[(int64_t)sess * p.b.max_rows_per_sess + g / p.grp];
        const int qh = h * p.grp + g % p.grp;
        v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)r * p.nq + qh) * HD + c * 8);
      }
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(qs + swz256(g, c)), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w));
    }
  }
  __syncthreads();
  const int total = s_total;
  const int k0 = (int)((int64_t)rank * total / C), k1 = (int)((int64_t)(rank + 1) * total / C);
  const int np = k1 - k0;

  auto meta = [&](int k) -> PageMeta {
    PageMeta m;
    if (k < s_ps) {
      m.page = p.b.sess_pages[(int64_t)sess * p.b.max_sess_pages + k];
      m.limit = min(PT, s_ls - k * PT);
      m.owner = -1;
    } else {
      int i = 0;
      while (k >= s_pstart[i + 1]) ++i;
      const int j = k - s_pstart[i];
      m.page = p.b.row_pages[(int64_t)s_rows[i] * p.b.max_row_pages + j];
      m.limit = min(PT, s_plen[i] - j * PT);
      m.owner = i;
    }
    return m;
  };

  const uint32_t ring = smem_u32(smem);
  if (warp == CW) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int j = 0; j < np; ++j) {
        const int st = j % NST;
        tma::mbar_wait(&empty[st], ((j / NST) & 1) ^ 1);
        const PageMeta m = meta(k0 + j);
        const int row_k = (int)((((int64_t)m.page * p.kv.n_layers + p.layer) * 2 * nkv + h) * PT);
        const int row_v = row_k + nkv * PT;
        unsigned char* dst = smem + st * STAGE;
        tma::mbar_expect_tx(&full[st], STAGE);
        tma::load_2d(&kvmap, &full[st], dst, 0, row_k);
        tma::load_2d(&kvmap, &full[st], dst + 2048, 64, row_k);
        tma::load_2d(&kvmap, &full[st], dst + TILE, 0, row_v);
        tma::load_2d(&kvmap, &full[st], dst + TILE + 2048, 64, row_v);
      }
    }
  }

  const int tile = warp / ways, way = warp % ways;
  const bool active = warp < CW && tile < T;
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  const int gA = tile * 16 + (lane >> 2), gB = gA + 8;
  if (active) {
    uint32_t qa[8][4];
    {
      const uint32_t qs = smem_u32(smem + OFF_Q);
      const int mi = lane >> 3;
      const int row = tile * 16 + (mi & 1) * 8 + (lane & 7);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        ldmatrix_x4(qs + swz256(row, 2 * ks + (mi >> 1)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    const int ownA = gA < G ? gA / p.grp : -2, ownB = gB < G ? gB / p.grp : -2;
    for (int j = way; j < np; j += ways) {
      const int st = j % NST;
      const PageMeta m = meta(k0 + j);
      tma::mbar_wait(&full[st], (j / NST) & 1);
      const uint32_t kt = ring + st * STAGE, vt = kt + TILE;
      float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      {
        const int mi = lane >> 3, ri = lane & 7;
        const int tok = (mi >> 1) * 8 + ri;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4(tile_addr(kt, tok, 2 * ks + (mi & 1)), b0, b1, b2, b3);
          mma_bf16_16816(s[0], qa[ks], b0, b1);
          mma_bf16_16816(s[1], qa[ks], b2, b3);
        }
      }
      const bool okA = m.owner < 0 || m.owner == ownA;
      const bool okB = m.owner < 0 || m.owner == ownB;
      const int cb = (lane & 3) * 2;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int t = nt * 8 + cb + (e & 1);
          const bool ok = t < m.limit && (e < 2 ? okA : okB);
          s[nt][e] = ok ? s[nt][e] * p.scale_log2 : -INFINITY;
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
        for (int np2 = 0; np2 < 8; ++np2) {
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4_trans(tile_addr(vt, tok, 2 * np2 + (mi >> 1)), b0, b1, b2, b3);
          mma_bf16_16816(o[2 * np2], pa, b0, b1);
          mma_bf16_16816(o[2 * np2 + 1], pa, b2, b3);
        }
      }
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&empty[st]);
    }
    l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
    l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
    l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  }
  __syncthreads();  // ring drained: every fetched page was consumed

  // -- fold the `ways` warps of each m-tile (ring reused as scratch)
  float* wO = reinterpret_cast<float*>(smem);       // [CW][16][HD+4]
  float* wM = wO + CW * 16 * (HD + 4);              // [CW][16]
  float* wL = wM + CW * 16;
  constexpr int LD = HD + 4;                        // padded row: conflict-free fragment stores
  if (active) {
    const int ra = lane >> 2, rb = ra + 8, cb = (lane & 3) * 2;
    float* w = wO + warp * 16 * LD;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      *reinterpret_cast<float2*>(w + ra * LD + nt * 8 + cb) = make_float2(o[nt][0], o[nt][1]);
      *reinterpret_cast<float2*>(w + rb * LD + nt * 8 + cb) = make_float2(o[nt][2], o[nt][3]);
    }
    if ((lane & 3) == 0) {
      wM[warp * 16 + ra] = m0;
      wM[warp * 16 + rb] = m1;
      wL[warp * 16 + ra] = l0;
      wL[warp * 16 + rb] = l1;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < T * 16 * HD; e += THREADS) {
    const int t = e / (16 * HD), rr = (e / HD) % 16, d = e % HD;
    float M = -INFINITY;
    for (int w = 0; w < ways; ++w) M = fmaxf(M, wM[(t * ways + w) * 16 + rr]);
    const float Mr = M == -INFINITY ? 0.f : M;
    float acc = 0.f, ls = 0.f;
    for (int w = 0; w < ways; ++w) {
      const int ww = t * ways + w;
      const float f = exp2f(wM[ww * 16 + rr] - Mr);
      acc += f * wO[(ww * 16 + rr) * LD + d];
      ls += f * wL[ww * 16 + rr];
    }
    const int g = t * 16 + rr;
    sO[g * HD + d] = acc;
    if (d == 0) {
      sM[g] = M;
      sL[g] = ls;
    }
  }

  // -- reduce the C CTA partials of the cluster through DSMEM
  tma::cluster_sync();
  const int E = G * HD;
  const int e0 = (int)((int64_t)rank * E / C), e1 = (int)((int64_t)(rank + 1) * E / C);
  for (int e = e0 + threadIdx.x; e < e1; e += THREADS) {
    const int g = e / HD, d = e % HD;
    float mc[C], lc[C], oc[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
      mc[c] = tma::ld_dsmem_f32(tma::map_rank(&sM[g], c));
      lc[c] = tma::ld_dsmem_f32(tma::map_rank(&sL[g], c));
      oc[c] = tma::ld_dsmem_f32(tma::map_rank(&sO[g * HD + d], c));
    }
    float M = -INFINITY;
#pragma unroll
    for (int c = 0; c < C; ++c) M = fmaxf(M, mc[c]);
    const float Mr = M == -INFINITY ? 0.f : M;
    float acc = 0.f, ls = 0.f;
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const float f = exp2f(mc[c] - Mr);
      acc += f * oc[c];
      ls += f * lc[c];
    }
    const int r = s_rows[g / p.grp];
    const int qh = h * p.grp + g % p.grp;
    p.out[((int64_t)r * p.nq + qh) * HD + d] = f2bf(ls > 0.f ? acc / ls : 0.f);
  }
  tma::cluster_sync();  // keep our shared memory alive until every peer is done reading it
}

// ------------------------------------------------------------ host side --

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static int kv_map(const psk_kv_layout& kv, CUtensorMap* out) {
  // one-entry cache keyed by the pool geometry
  static CUtensorMap cached;
  static psk_kv_layout key = {};
  if (key.base == kv.base && key.n_pages == kv.n_pages && key.page_elems == kv.page_elems) {
    *out = cached;
    return PSK_OK;
  }
  static EncodeTiledFn enc = nullptr;
  if (!enc) {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PSK_ECUDA;
    }
    enc = reinterpret_cast<EncodeTiledFn>(fp);
  }
  const cuuint64_t rows = (cuuint64_t)kv.n_pages * (cuuint64_t)kv.page_elems / HD;
  cuuint64_t dims[2] = {(cuuint64_t)HD, rows};
  cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)PT};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&cached, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv.base, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("KV tensor map encode failed (%d)", (int)r);
    return PSK_ECUDA;
  }
  key = kv;
  *out = cached;
  return PSK_OK;
}

template <int C>
static int launch(const CUtensorMap& map, const Params& p, int n_clusters, cudaStream_t s) {
  static bool init = false;
  if (!init) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(decode_attn_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM));
    if (C > 8)
      PSK_CUDA_TRY(cudaFuncSetAttribute(decode_attn_kernel<C>,
                                        cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    init = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_clusters * C);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_attn_kernel<C>, map, p));
  return PSK_OK;
}

}  // namespace dattn
}  // namespace psk

extern "C" int psk_decode_attn(const psk_decode_batch* b, const void* q_rot, int32_t n_q_heads,
                               int32_t layer, psk_kv_layout kv, int32_t cluster, void* out,
                               void* stream) {
  using namespace psk::dattn;
  PSK_CHECK_ARG(b && q_rot && out && kv.head_dim == HD && kv.page_tokens == PT && kv.n_pages > 0 &&
                    n_q_heads % kv.n_kv_heads == 0,
                "psk_decode_attn: bad args");
  const int grp = n_q_heads / kv.n_kv_heads;
  PSK_CHECK_ARG(b->max_rows_per_sess <= MAXR && grp * b->max_rows_per_sess <= GMAX,
                "psk_decode_attn: %d query rows per KV head exceed %d", grp * b->max_rows_per_sess, GMAX);
  if (b->n_rows == 0) return PSK_OK;
  CUtensorMap map;
  int rc = kv_map(kv, &map);
  if (rc) return rc;
  Params p;
  p.b = *b;
  p.kv = kv;
  p.q = reinterpret_cast<const __nv_bfloat16*>(q_rot);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.nq = n_q_heads;
  p.grp = grp;
  p.layer = layer;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  const int nc = b->n_sess * kv.n_kv_heads;
  cudaStream_t s = psk::as_stream(stream);
  switch (cluster) {
    case 1: return launch<1>(map, p, nc, s);
    case 2: return launch<2>(map, p, nc, s);
    case 4: return launch<4>(map, p, nc, s);
    case 8: return launch<8>(map, p, nc, s);
    case 16: return launch<16>(map, p, nc, s);
    default:
      psk::set_error("psk_decode_attn: cluster must be 1, 2, 4, 8 or 16 (got %d)", cluster);
      return PSK_EINVAL;
  }
}
