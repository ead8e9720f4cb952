// K6 — shared-prefix paged decode attention (one layer per call).
//
// Decode modules batched on one session share the base module's prompt KV
// (the PrefillShare cache reuse: frontend/src/evaluate.ts:21-50, one base
// cache consumed by several decoders; the reference re-concatenates and
// re-reads the full past per model and per step, model.ts:307-315).
//
// Partial kernel: one CTA = (session, KV head, split). Its page stream is the
// split's slice of [shared prompt pages | row 0 private pages | row 1 private
// pages | ...]. A producer warp streams every page with TMA (one 4-D
// 128B-swizzled box = the page's 8 KiB of K and V for this head and layer)
// through a 16-stage (128 KiB) mbarrier ring; 8
// consumer warps map to (query m-tile, page subset), so each page is read
// from HBM once per step for ALL query rows of the session (GQA group x
// co-batched decode modules, <= 64 rows); private pages mask the rows they do
// not own. Warps fold their online-softmax state in fragment order, and the
// CTA writes one (m, l, O) partial per query row.
// A merge kernel (one thread per output element, all split partials in
// flight at once) folds the partials by log-sum-exp. Both kernels use
// programmatic dependent launch: the partial kernel's prologue (row and page
// tables) overlaps its producer (RoPE + KV append) and the merge launch
// overlaps the partial kernel's tail.
//
// (A 16-CTA-cluster / DSMEM-reduction variant was measured first: at this
// shared-memory footprint only 7 such clusters are co-resident on a B200, so
// 8 KV heads always ran in two waves.)
#include "common.cuh"
#include "mma.cuh"
#include "tma.cuh"

#include <math.h>

namespace psk {
namespace dattn {

constexpr int HD = 128, PT = 16;
constexpr int CW = 8;                   // consumer warps
constexpr int THREADS = (CW + 1) * 32;  // + 1 TMA producer warp
#ifndef PSK_ATTN_NST
#define PSK_ATTN_NST 16
#endif
constexpr int NST = PSK_ATTN_NST;       // pipeline stages (1 page = K + V each, 8 KiB)
constexpr int TILE = PT * HD * 2;       // 4 KiB
constexpr int STAGE = 2 * TILE;
constexpr int GMAX = 64;
constexpr int MAXR = 16;                // decode rows per session
constexpr int OFF_Q = NST * STAGE;
constexpr int OFF_BAR = OFF_Q + GMAX * 256;  // +16 KiB
constexpr int MAXP = 1024;              // page indices staged in smem
constexpr int OFF_PG = OFF_BAR + 2 * NST * 8;
constexpr int SMEM = OFF_PG + MAXP * 4 + 1024;  // ~150 KiB (+ alignment slack): 1 CTA / SM
constexpr int FRAG = 68;                // floats per lane in the fold scratch (64 O + m0 m1 l0 l1)
static_assert(CW * 32 * FRAG * 4 <= OFF_BAR, "fold scratch must fit in ring + Q");

struct Params {
  psk_decode_batch b;
  psk_kv_layout kv;
  const __nv_bfloat16* q;  // [rows][nq][HD]
  __nv_bfloat16* out;      // [rows][nq][HD]
  float* pm;               // [items][GMAX]
  float* pl;               // [items][GMAX]
  float* po;               // [items][GMAX][HD]
  int nq, grp, layer, ns;
  float scale_log2;
};

// SW128 address of (token row, 16-byte chunk c16 in 0..15) in a K/V tile made
// of two [16 x 128 B] TMA boxes (dims 0-63, 64-127).
__device__ __forceinline__ uint32_t tile_addr(uint32_t tile, int tok, int c16) {
  return tile + ((c16 >> 3) << 11) + tok * 128 + (((c16 & 7) ^ (tok & 7)) << 4);
}

__global__ void __launch_bounds__(THREADS, 1)
    decode_attn_partial(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* empty = full + NST;
  int* s_page = reinterpret_cast<int*>(smem + OFF_PG);
  __shared__ int s_rows[MAXR], s_plen[MAXR], s_pstart[MAXR + 1];
  __shared__ int s_ps, s_ls, s_total;

  trace_stamp(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  const int item = blockIdx.x;
  const int j_split = item % p.ns;
  const int h = (item / p.ns) % nkv;
  const int sess = item / (p.ns * nkv);
  const int nr = p.b.sess_nrows[sess];
  const int G = nr * p.grp;
  const int T = (G + 15) / 16;
  const int Tp = T <= 1 ? 1 : (T == 2 ? 2 : 4);
  const int ways = CW / Tp;

  // prologue: one latency round trip for all rows (no dependent chains)
  if (threadIdx.x < nr) {
    const int r = p.b.sess_rows[(int64_t)sess * p.b.max_rows_per_sess + threadIdx.x];
    s_rows[threadIdx.x] = r;
    s_plen[threadIdx.x] = p.b.priv_len[r] + 1;  // includes the token appended this step
  } else if (threadIdx.x == 32) {
    s_ls = p.b.sess_len[sess];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int Ps = (s_ls + PT - 1) / PT;
    s_ps = Ps;
    int acc = Ps;
    for (int i = 0; i < nr; ++i) {
      s_pstart[i] = acc;
      acc += (s_plen[i] + PT - 1) / PT;
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
  __syncthreads();
  trace_stamp(1);
  const int total = s_total;
  const int k0 = (int)((int64_t)j_split * total / p.ns);
  const int k1 = (int)((int64_t)(j_split + 1) * total / p.ns);
  const int np = k1 - k0;

  auto page_of = [&](int k) -> int {
    if (k < s_ps) return p.b.sess_pages[(int64_t)sess * p.b.max_sess_pages + k];
    int i = 0;
    while (k >= s_pstart[i + 1]) ++i;
    return p.b.row_pages[(int64_t)s_rows[i] * p.b.max_row_pages + (k - s_pstart[i])];
  };
  // page indices -> shared memory (tables are static within a step)
  for (int j = threadIdx.x; j < np && j < MAXP; j += THREADS) s_page[j] = page_of(k0 + j);
  // everything above overlaps the producer of q / the new K,V (PDL)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  {
    const uint32_t qs = smem_u32(smem + OFF_Q);
    for (int e = threadIdx.x; e < T * 16 * 16; e += THREADS) {
      const int g = e >> 4, c = e & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (g < G) {
        const int qh = h * p.grp + g % p.grp;
        v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)s_rows[g / p.grp] * p.nq + qh) * HD + c * 8);
      }
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(qs + swz256(g, c)), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w));
    }
  }
  __syncthreads();
  trace_stamp(2);

  const uint32_t ring = smem_u32(smem);
  if (warp == CW) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      for (int j = 0; j < np; ++j) {
        const int st = j % NST;
        tma::mbar_wait(&empty[st], ((j / NST) & 1) ^ 1);
        const int page = j < MAXP ? s_page[j] : page_of(k0 + j);
        const int row_k = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv + h) * PT);
        tma::mbar_expect_tx(&full[st], STAGE);
        tma::load_4d(&kvmap, &full[st], smem + st * STAGE, 0, row_k, 0, 0);  // K and V, 8 KiB
      }
    }
  }

  const int tile = warp / ways, way = warp % ways;
  const bool active = warp < CW && tile < T;
  float o[16][4];
#pragma unroll
  for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  if (active) {
    uint32_t qa[8][4];
    {
      const uint32_t qs = smem_u32(smem + OFF_Q);
      const int qrow = tile * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks)
        ldmatrix_x4(qs + swz256(qrow, 2 * ks + (lane >> 4)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
    }
    const int gA = tile * 16 + (lane >> 2), gB = gA + 8;
    const int ownA = gA < G ? gA / p.grp : -2, ownB = gB < G ? gB / p.grp : -2;
    for (int j = way; j < np; j += ways) {
      const int st = j % NST;
      int limit, owner;
      {
        const int k = k0 + j;
        if (k < s_ps) {
          limit = min(PT, s_ls - k * PT);
          owner = -1;
        } else {
          int i = 0;
          while (k >= s_pstart[i + 1]) ++i;
          limit = min(PT, s_plen[i] - (k - s_pstart[i]) * PT);
          owner = i;
        }
      }
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
      const bool okA = owner < 0 || owner == ownA;
      const bool okB = owner < 0 || owner == ownB;
      const int cb = (lane & 3) * 2;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int t = nt * 8 + cb + (e & 1);
          const bool ok = t < limit && (e < 2 ? okA : okB);
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
  trace_stamp(3);
  asm volatile("griddepcontrol.launch_dependents;");

  // -- fold the `ways` warps of each m-tile in fragment order (ring + Q reused)
  float* scr = reinterpret_cast<float*>(smem);  // [CW][32][FRAG]
  if (active) {
    float4* d = reinterpret_cast<float4*>(scr + (warp * 32 + lane) * FRAG);
#pragma unroll
    for (int i = 0; i < 16; ++i) d[i] = make_float4(o[i][0], o[i][1], o[i][2], o[i][3]);
    d[16] = make_float4(m0, m1, l0, l1);
  }
  __syncthreads();
  const int64_t base = (int64_t)item * GMAX;
  // thread (warp w, lane l) owns fragment elements [8w, 8w+8) of lane l, per tile
  if (warp < CW) {
    const int ra = lane >> 2, rb = ra + 8, cb = (lane & 3) * 2;
    for (int t = 0; t < T; ++t) {
      float Ma = -INFINITY, Mb = -INFINITY;
      for (int v = 0; v < ways; ++v) {
        const float4 ml = reinterpret_cast<const float4*>(scr + ((t * ways + v) * 32 + lane) * FRAG)[16];
        Ma = fmaxf(Ma, ml.x);
        Mb = fmaxf(Mb, ml.y);
      }
      const float Mra = Ma == -INFINITY ? 0.f : Ma, Mrb = Mb == -INFINITY ? 0.f : Mb;
      float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
      float La = 0.f, Lb = 0.f;
      for (int v = 0; v < ways; ++v) {
        const float* src = scr + ((t * ways + v) * 32 + lane) * FRAG;
        const float4 ml = reinterpret_cast<const float4*>(src)[16];
        const float fa = exp2f(ml.x - Mra), fb = exp2f(ml.y - Mrb);
        La += fa * ml.z;
        Lb += fb * ml.w;
        const float4 x0 = reinterpret_cast<const float4*>(src)[2 * warp];
        const float4 x1 = reinterpret_cast<const float4*>(src)[2 * warp + 1];
        acc[0] += fa * x0.x; acc[1] += fa * x0.y; acc[2] += fb * x0.z; acc[3] += fb * x0.w;
        acc[4] += fa * x1.x; acc[5] += fa * x1.y; acc[6] += fb * x1.z; acc[7] += fb * x1.w;
      }
      const int ga = t * 16 + ra, gb = t * 16 + rb;
      // elements 8w..8w+7 = fragments nt = 2w, 2w+1; each (a0 a1 b0 b1)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int col = (2 * warp + q) * 8 + cb;
        if (ga < G)
          *reinterpret_cast<float2*>(p.po + (base + ga) * HD + col) = make_float2(acc[4 * q], acc[4 * q + 1]);
        if (gb < G)
          *reinterpret_cast<float2*>(p.po + (base + gb) * HD + col) = make_float2(acc[4 * q + 2], acc[4 * q + 3]);
      }
      if (warp == 0 && (lane & 3) == 0) {
        if (ga < G) {
          p.pm[base + ga] = Ma;
          p.pl[base + ga] = La;
        }
        if (gb < G) {
          p.pm[base + gb] = Mb;
          p.pl[base + gb] = Lb;
        }
      }
    }
  }

  trace_stamp(4);
}

// Merge: one CTA per (row, q head), one thread per head dim; every split's
// (m, l, o) is loaded up front (32 splits in flight per thread) and folded by
// log-sum-exp. Launched with programmatic dependent launch: it is scheduled
// while the partial kernel drains and waits on griddepcontrol for its data.
constexpr int MERGE_U = 32;
__global__ void __launch_bounds__(HD) decode_attn_merge(const __grid_constant__ Params p) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");  // the o-proj GEMV may start streaming weights
  const int r = blockIdx.x, qh = blockIdx.y, d = threadIdx.x;
  const int nkv = p.kv.n_kv_heads;
  const int h = qh / p.grp;
  const int g = p.b.row_in_sess[r] * p.grp + qh % p.grp;
  const int64_t base = (int64_t)(p.b.row_sess[r] * nkv + h) * p.ns * GMAX + g;
  float M = -INFINITY, L = 0.f, acc = 0.f;
  for (int j0 = 0; j0 < p.ns; j0 += MERGE_U) {
    float mj[MERGE_U], lj[MERGE_U], oj[MERGE_U];
#pragma unroll
    for (int u = 0; u < MERGE_U; ++u) {
      const int j = j0 + u;
      const int64_t sl = base + (int64_t)j * GMAX;
      const bool ok = j < p.ns;
      mj[u] = ok ? __ldcg(p.pm + sl) : -INFINITY;
      lj[u] = ok ? __ldcg(p.pl + sl) : 0.f;
      oj[u] = ok ? __ldcg(p.po + sl * HD + d) : 0.f;
    }
    float Mc = M;
#pragma unroll
    for (int u = 0; u < MERGE_U; ++u) Mc = fmaxf(Mc, mj[u]);
    const float Mr = Mc == -INFINITY ? 0.f : Mc;
    const float a = exp2f(M - Mr);
    L *= a;
    acc *= a;
#pragma unroll
    for (int u = 0; u < MERGE_U; ++u) {
      const float f = exp2f(mj[u] - Mr);
      L += f * lj[u];
      acc += f * oj[u];
    }
    M = Mc;
  }
  p.out[((int64_t)r * p.nq + qh) * HD + d] = f2bf(L > 0.f ? acc / L : 0.f);
}

// ------------------------------------------------- tcgen05 fan-out path ----
// When a session carries many decode rows (fan-out: up to 16 modules x 4 GQA
// heads = 64 query rows per KV head) the mma.sync kernel above is bound by
// the legacy tensor pipe, not HBM. This variant runs both products on the
// 5th-gen tensor cores: per 8-page chunk (128 tokens),
//   S[128 rows x 128 tok] = Q . K^T   (8 UMMA M=128 N=128 K=16, TMEM)
//   D[128 rows x 128 dim] = P . V     (8 UMMA, V as an MN-major B operand)
// A producer warp streams K/V chunks with TMA into a 2-stage ring (K boxes
// laid out so the chunk's 128 token rows sit at a uniform 128 B stride), an
// MMA warp issues tcgen05.mma, and 4 softmax warps own one query row each
// (thread = TMEM lane): they read S, write bf16 P back to shared memory in
// the UMMA K-major SW128 layout, and fold D into an fp32 O held in
// registers with the online-softmax rescale.
namespace tcv {

constexpr int CP = 8;                  // pages per chunk
constexpr int NSTG = 2;                // chunk stages
constexpr int KREG = CP * TILE;        // 32 KiB: [dims 0-63 box x 8 pages][dims 64-127 box x 8 pages]
constexpr int VREG = CP * TILE;        // 32 KiB: [page][box0 | box1]
constexpr int STG = KREG + VREG;
constexpr int OFF_Q = NSTG * STG;      // 128 KiB
constexpr int OFF_P = OFF_Q + 32768;   // Q: [2 boxes][128 rows][128 B]
constexpr int OFF_BAR = OFF_P + 32768; // P: same layout
constexpr int OFF_PG = OFF_BAR + 256;
constexpr int SMEM = OFF_PG + MAXP * 4 + 1024;
constexpr int THREADS = 192;           // w0 TMA, w1 MMA (+TMEM alloc), w2-5 softmax
constexpr int TMEM_COLS = 256;         // S: cols [0,128), D: cols [128,256)

__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// MN-major SW128: 64-element MN groups at LBO, 8-row K groups at SBO.
__device__ __forceinline__ uint64_t desc_mn_sw128(uint32_t addr, uint32_t lbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(1024 >> 4) << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(bool b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(128 >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   tma::sa(bar))
               : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
        "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
        "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__global__ void __launch_bounds__(THREADS, 1)
    decode_attn_tc(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* full = bars;            // [2]
  uint64_t* empty = bars + 2;       // [2]
  uint64_t* s_full = bars + 4;
  uint64_t* s_empty = bars + 5;
  uint64_t* p_full = bars + 6;
  uint64_t* d_full = bars + 7;
  uint64_t* d_empty = bars + 8;
  int* s_page = reinterpret_cast<int*>(smem + OFF_PG);
  __shared__ int s_rows[MAXR], s_plen[MAXR], s_pstart[MAXR + 1];
  __shared__ int s_ps, s_ls, s_total;
  __shared__ uint32_t s_tmem;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads;
  const int item = blockIdx.x;
  const int j_split = item % p.ns;
  const int h = (item / p.ns) % nkv;
  const int sess = item / (p.ns * nkv);
  const int nr = p.b.sess_nrows[sess];
  const int G = nr * p.grp;

  if (threadIdx.x < nr) {
    const int r = p.b.sess_rows[(int64_t)sess * p.b.max_rows_per_sess + threadIdx.x];
    s_rows[threadIdx.x] = r;
    s_plen[threadIdx.x] = p.b.priv_len[r] + 1;
  } else if (threadIdx.x == 32) {
    s_ls = p.b.sess_len[sess];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const int Ps = (s_ls + PT - 1) / PT;
    s_ps = Ps;
    int acc = Ps;
    for (int i = 0; i < nr; ++i) {
      s_pstart[i] = acc;
      acc += (s_plen[i] + PT - 1) / PT;
    }
    s_pstart[nr] = acc;
    s_total = acc;
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
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tma::sa(&s_tmem)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  __syncthreads();
  const int total = s_total;
  const int k0 = (int)((int64_t)j_split * total / p.ns);
  const int k1 = (int)((int64_t)(j_split + 1) * total / p.ns);
  const int np = k1 - k0;
  const int nch = (np + CP - 1) / CP;
  for (int j = threadIdx.x; j < np && j < MAXP; j += THREADS) {
    const int k = k0 + j;
    int pg;
    if (k < s_ps) {
      pg = p.b.sess_pages[(int64_t)sess * p.b.max_sess_pages + k];
    } else {
      int i = 0;
      while (k >= s_pstart[i + 1]) ++i;
      pg = p.b.row_pages[(int64_t)s_rows[i] * p.b.max_row_pages + (k - s_pstart[i])];
    }
    s_page[j] = pg;
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // Q -> shared, UMMA K-major SW128: [box = dims/64][row][128 B], rows >= G zero
  for (int e = threadIdx.x; e < 128 * 16; e += THREADS) {
    const int g = e >> 4, c = e & 15;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (g < G) {
      const int qh = h * p.grp + g % p.grp;
      v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)s_rows[g / p.grp] * p.nq + qh) * HD + c * 8);
    }
    const uint32_t a = smem_u32(smem + OFF_Q) + (c >> 3) * 16384 + g * 128 + (((c & 7) ^ (g & 7)) << 4);
    asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t sq = smem_u32(smem + OFF_Q), sp = smem_u32(smem + OFF_P);

  if (warp == 0) {
    if (lane == 0 && np > 0) {
      for (int c = 0; c < nch; ++c) {
        const int st = c % NSTG;
        tma::mbar_wait(&empty[st], ((c / NSTG) & 1) ^ 1);
        tma::mbar_expect_tx(&full[st], STG);
        unsigned char* kr = smem + st * STG;
        unsigned char* vr = kr + KREG;
        for (int pp = 0; pp < CP; ++pp) {
          const int j = c * CP + pp;
          // pages past the slice reload a valid page (finite data); masked below
          const int jj = j < np ? j : c * CP;
          const int page = jj < MAXP ? s_page[jj] : s_page[0];
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
    if (lane == 0 && np > 0) {
      constexpr uint32_t ID_QK = idesc(false), ID_PV = idesc(true);
      for (int c = 0; c < nch; ++c) {
        const int st = c % NSTG;
        const uint32_t kr = smem_u32(smem + st * STG), vr = kr + KREG;
        tma::mbar_wait(&full[st], (c / NSTG) & 1);
        tma::mbar_wait(s_empty, (c & 1) ^ 1);
        fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint64_t a = desc_k_sw128(sq + (kk >> 2) * 16384) + 2 * (kk & 3);
          const uint64_t b = desc_k_sw128(kr + (kk >> 2) * (CP * 2048)) + 2 * (kk & 3);
          umma(tmem, a, b, ID_QK, kk > 0);
        }
        commit(s_full);
        tma::mbar_wait(p_full, c & 1);
        tma::mbar_wait(d_empty, (c & 1) ^ 1);
        fence_after();
#pragma unroll
        for (int pp = 0; pp < CP; ++pp) {
          const uint64_t a = desc_k_sw128(sp + (pp >> 2) * 16384) + 2 * (pp & 3);
          const uint64_t b = desc_mn_sw128(vr + pp * TILE, 2048);
          umma(tmem + 128, a, b, ID_PV, pp > 0);
        }
        commit(d_full);
        commit(&empty[st]);
      }
    }
  } else {
    // ---------------- softmax: thread = query row = TMEM lane ----------------
    const int q = warp & 3;
    const int g = q * 32 + lane;
    const uint32_t tS = tmem + ((uint32_t)(q * 32) << 16);
    const uint32_t tD = tS + 128;
    const int own = g < G ? g / p.grp : -2;
    float O[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) O[i] = 0.f;
    float m = -INFINITY, l = 0.f;
    for (int c = 0; c < nch; ++c) {
      int lim[CP], ownr[CP];
#pragma unroll
      for (int pp = 0; pp < CP; ++pp) {
        const int j = c * CP + pp;
        const int k = k0 + j;
        if (j >= np) {
          lim[pp] = 0;
          ownr[pp] = -1;
        } else if (k < s_ps) {
          lim[pp] = min(PT, s_ls - k * PT);
          ownr[pp] = -1;
        } else {
          int i = 0;
          while (k >= s_pstart[i + 1]) ++i;
          lim[pp] = min(PT, s_plen[i] - (k - s_pstart[i]) * PT);
          ownr[pp] = i;
        }
        if (ownr[pp] >= 0 && ownr[pp] != own) lim[pp] = 0;
      }
      tma::mbar_wait(s_full, c & 1);
      fence_after();
      float mx = -INFINITY;
      float v[32];
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        ld32(tS + gi * 32, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const int col = gi * 32 + e;
          if ((col & 15) < lim[col >> 4]) mx = fmaxf(mx, v[e] * p.scale_log2);
        }
      }
      const float mn = fmaxf(m, mx);
      const float base = mn == -INFINITY ? 0.f : mn;
      const float alpha = exp2f(m - base);
      float ladd = 0.f;
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        ld32(tS + gi * 32, v);
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int col = gi * 32 + e;
          const float p0 = (col & 15) < lim[col >> 4] ? exp2f(v[e] * p.scale_log2 - base) : 0.f;
          const float p1 = ((col + 1) & 15) < lim[(col + 1) >> 4] ? exp2f(v[e + 1] * p.scale_log2 - base) : 0.f;
          ladd += p0 + p1;
          pk[e >> 1] = pack_bf16(p0, p1);
        }
        // 32 tokens = 4 16-byte chunks of this row; K-major SW128 like Q
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) {
          const int chunk = gi * 4 + cc;  // 0..15 (8 tokens each)
          const uint32_t a = sp + (chunk >> 3) * 16384 + g * 128 + (((chunk & 7) ^ (g & 7)) << 4);
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(pk[4 * cc]), "r"(pk[4 * cc + 1]),
                       "r"(pk[4 * cc + 2]), "r"(pk[4 * cc + 3]));
        }
      }
      fence_before();
      tma::mbar_arrive(s_empty);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tma::mbar_arrive(p_full);
      l = l * alpha + ladd;
      tma::mbar_wait(d_full, c & 1);
      fence_after();
#pragma unroll
      for (int gi = 0; gi < 4; ++gi) {
        ld32(tD + gi * 32, v);
#pragma unroll
        for (int e = 0; e < 32; ++e) O[gi * 32 + e] = O[gi * 32 + e] * alpha + v[e];
      }
      fence_before();
      tma::mbar_arrive(d_empty);
      m = mn;
    }
    if (g < G) {
      const int64_t slot = (int64_t)item * GMAX + g;
      p.pm[slot] = m;
      p.pl[slot] = l;
      float4* dst = reinterpret_cast<float4*>(p.po + slot * HD);
#pragma unroll
      for (int i = 0; i < HD / 4; ++i) dst[i] = make_float4(O[4 * i], O[4 * i + 1], O[4 * i + 2], O[4 * i + 3]);
    }
  }
  fence_before();
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  if (warp == 1) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TMEM_COLS));
  }
}

}  // namespace tcv

// ------------------------------------------------------------ host side --

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

}  // namespace dattn

// 2D TMA map over a KV page pool: rows of 128 dims (256 B), [16 x 64] boxes,
// 128B swizzle. Cached per pool geometry. Shared by the attention kernels.
int kv_tensor_map(const psk_kv_layout& kv, CUtensorMap* out, bool page_box) {
  using namespace dattn;
  // small cache keyed by the pool geometry and the box kind
  static CUtensorMap cached[8];
  static psk_kv_layout keys[8] = {};
  static bool kinds[8] = {};
  static int next = 0;
  for (int i = 0; i < 8; ++i)
    if (keys[i].base == kv.base && keys[i].n_pages == kv.n_pages && keys[i].page_elems == kv.page_elems &&
        kinds[i] == page_box) {
      *out = cached[i];
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
  const int i = next;
  next = (next + 1) % 8;
  CUresult r;
  if (!page_box) {
    cuuint64_t dims[2] = {(cuuint64_t)HD, rows};
    cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)PT};
    cuuint32_t es[2] = {1, 1};
    r = enc(&cached[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv.base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // (dim, token row, half, K|V): the V tile of a (page, layer, head) sits
    // n_kv_heads tiles after its K tile
    cuuint64_t dims[4] = {64, rows, 2, 2};
    cuuint64_t strides[3] = {(cuuint64_t)HD * 2, 128, (cuuint64_t)kv.n_kv_heads * PT * HD * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)PT, 2, 2};
    cuuint32_t es[4] = {1, 1, 1, 1};
    r = enc(&cached[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, kv.base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  if (r != CUDA_SUCCESS) {
    keys[i] = psk_kv_layout{};
    set_error("KV tensor map encode failed (%d)", (int)r);
    return PSK_ECUDA;
  }
  keys[i] = kv;
  kinds[i] = page_box;
  *out = cached[i];
  return PSK_OK;
}

}  // namespace psk

using namespace psk::dattn;

extern "C" {

int psk_decode_attn_workspace(const psk_decode_batch* b, int32_t n_kv_heads, int32_t splits,
                              int64_t* bytes) {
  PSK_CHECK_ARG(b && bytes && splits >= 1, "psk_decode_attn_workspace: bad args");
  const int64_t items = (int64_t)b->n_sess * n_kv_heads * splits;
  *bytes = items * GMAX * (HD + 2) * 4;
  return PSK_OK;
}

int psk_decode_attn(const psk_decode_batch* b, const void* q_rot, int32_t n_q_heads, int32_t layer,
                    psk_kv_layout kv, int32_t splits, void* workspace, void* out, void* stream) {
  PSK_CHECK_ARG(b && q_rot && out && workspace && kv.head_dim == HD && kv.page_tokens == PT &&
                    kv.n_pages > 0 && n_q_heads % kv.n_kv_heads == 0 && splits >= 1,
                "psk_decode_attn: bad args");
  const int grp = n_q_heads / kv.n_kv_heads;
  PSK_CHECK_ARG(b->max_rows_per_sess <= MAXR && grp * b->max_rows_per_sess <= GMAX,
                "psk_decode_attn: %d query rows per KV head exceed %d", grp * b->max_rows_per_sess, GMAX);
  if (b->n_rows == 0) return PSK_OK;
  // tcgen05 fan-out path: opt-in (PSK_ATTN_TC=1) until it beats mma.sync —
  // measured on B200 it does not yet (32k x 16 modules: 100 us vs 51 us)
  static const bool use_tc_env = getenv("PSK_ATTN_TC") != nullptr;
  const bool use_tc = grp * b->max_rows_per_sess > 16 && use_tc_env;
  CUtensorMap map;
  int rc = psk::kv_tensor_map(kv, &map, /*page_box=*/!use_tc);
  if (rc) return rc;
  Params p;
  p.b = *b;
  p.kv = kv;
  p.q = reinterpret_cast<const __nv_bfloat16*>(q_rot);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.nq = n_q_heads;
  p.grp = grp;
  p.layer = layer;
  p.ns = splits;
  const int64_t items = (int64_t)b->n_sess * kv.n_kv_heads * splits;
  float* ws = reinterpret_cast<float*>(workspace);
  p.pm = ws;
  p.pl = ws + items * GMAX;
  p.po = ws + 2 * items * GMAX;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  cudaStream_t s = psk::as_stream(stream);
  static bool init = false;
  if (!init) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(decode_attn_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM));
    init = true;
  }
  const bool tr = psk::trace_arm((int)items);
  cudaLaunchAttribute pdl[1];
  pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  pdl[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)items);
  cfg.stream = s;
  cfg.attrs = pdl;
  cfg.numAttrs = 1;
  if (use_tc) {
    static bool tc_init = false;
    if (!tc_init) {
      PSK_CUDA_TRY(cudaFuncSetAttribute(tcv::decode_attn_tc, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        tcv::SMEM));
      tc_init = true;
    }
    cfg.blockDim = dim3(tcv::THREADS);
    cfg.dynamicSmemBytes = tcv::SMEM;
    PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, tcv::decode_attn_tc, map, p));
  } else {
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM;
    PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_attn_partial, map, p));
  }
  if (tr) {
    static const char* names[] = {"entry", "prologue", "staged", "loop-done", "folded"};
    psk::trace_report("decode_attn", (int)items, 5, names);
    psk::trace_disarm();
  }
  cudaLaunchConfig_t mcfg = {};
  mcfg.gridDim = dim3(b->n_rows, n_q_heads);
  mcfg.blockDim = dim3(HD);
  mcfg.stream = s;
  mcfg.attrs = pdl;
  mcfg.numAttrs = 1;
  PSK_CUDA_TRY(cudaLaunchKernelEx(&mcfg, decode_attn_merge, p));

  return PSK_OK;
}

}  // extern "C"
