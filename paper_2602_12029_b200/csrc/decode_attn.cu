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
#include "umma.cuh"

#include <math.h>

namespace psk {
namespace dattn {

constexpr int HD = 128, PT = 16;
constexpr int CW = 8;                   // consumer warps
constexpr int THREADS = (CW + 1) * 32;  // + 1 TMA producer warp
#ifndef PSK_ATTN_NST
#define PSK_ATTN_NST 16
#endif
constexpr int NST = PSK_ATTN_NST;
#ifndef PSK_ATTN_EARLY
#define PSK_ATTN_EARLY 0  // 1: the TMA producer streams shared pages before the PDL wait (measured slower: 4k x 8 sessions 36.7 -> 43.9 us)
#endif       // pipeline stages (1 page = K + V each, 8 KiB)
constexpr int TILE = PT * HD * 2;       // 4 KiB
constexpr int STAGE = 2 * TILE;
constexpr int GMAX = 64;
constexpr int CNT_INTS = 8192;          // workspace head: fused-merge words (2 ints per group)
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
  int* dir;  // stream-K mode (ns == 0): per group {first CTA, last CTA}, then the page total;
             // partial slot of (cta, group) = cta + group
  int sk_grid;  // stream-K: CTAs of the partial kernel
  unsigned* cnt;  // fan-out kernel, fused merge: per group generation << 16 | arrivals (+ a spare word)
  int fused;      // fan-out kernel: the split CTAs merge their group themselves (no merge kernel)
  int early;      // fan-out kernel: stream shared pages before the PDL wait (default; PSK_ATTN_LATE=1: off)
  int stream_only;  // fan-out kernel, measurement only (PSK_ATTN_STREAM_ONLY=1): pages streamed and
                    // released without MMA / softmax (the TMA stream's own ceiling; output garbage)
  unsigned long long* ring;  // fan-out kernel, diagnostics (PSK_TRACE_RING=1): this launch's slot of
                             // per-CTA %globaltimer stamps, 8 per CTA (nullptr: off)
};

// In-kernel split merge barrier (the split CTAs of a group are co-resident:
// grid <= SMs, 1 CTA per SM). One word per group: generation << 16 |
// arrivals. The last arrival adds (1 << 16) - ns (next generation, arrivals
// back to 0); the others wait for the generation to move past the one their
// arrival saw. A CTA releases its PDL dependents only after its arrival, so a
// back-to-back launch of the kernel never reaches the word before every
// arrival of this launch (and its generation step) is in: no reset pass and
// no departure count. Call with the CTA's partial written (all threads).
__device__ __forceinline__ void split_barrier(unsigned* word, unsigned ns) {
  __shared__ unsigned s_target;
  __syncthreads();  // this CTA's partial is written
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned old = atomicAdd(word, 1u);
    if ((old & 0xffffu) == ns - 1) atomicAdd(word, 0x10000u - ns);
    s_target = ((old >> 16) + 1u) & 0xffffu;
  }
  __syncthreads();
  asm volatile("griddepcontrol.launch_dependents;");
  if (threadIdx.x == 0) {
    unsigned v;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(word) : "memory");
    } while ((short)((v >> 16) - s_target) < 0);
    __threadfence();
  }
}

// Launch-ring stamp (thread 0 of the CTA = the producer warp's lane 0)
__device__ __forceinline__ void ring_stamp(const Params& p, int k) {
  if (p.ring != nullptr && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    p.ring[(size_t)blockIdx.x * 8 + k] = v;
  }
}

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
  __syncthreads();
  // Everything above overlaps the producer of q / the new K,V (PDL). The TMA
  // producer streams the shared prompt pages without waiting: only q and the
  // private pages (which hold this step's appended token) come from
  // rope_append; no kernel of a decode step writes shared pages.
  if (warp < CW) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const uint32_t qs = smem_u32(smem + OFF_Q);
    for (int e = threadIdx.x; e < T * 16 * 16; e += CW * 32) {
      const int g = e >> 4, c = e & 15;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (g < G) {
        const int qh = h * p.grp + g % p.grp;
        v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)s_rows[g / p.grp] * p.nq + qh) * HD + c * 8);
      }
      asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(qs + swz256(g, c)), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w));
    }
    named_barrier_sync(1, CW * 32);  // Q staged (consumer warps only)
  }
  trace_stamp(2);

  const uint32_t ring = smem_u32(smem);
  if (warp == CW) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      bool dep = false;
      for (int j = 0; j < np; ++j) {
        const int st = j % NST;
        if (!dep && (k0 + j >= s_ps || !PSK_ATTN_EARLY)) {  // first private page: wait for rope_append
          asm volatile("griddepcontrol.wait;" ::: "memory");
          dep = true;
        }
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


// ------------------------------------------------ stream-K partial kernel --
// The (session, KV head) groups of a step have very different page counts
// (shared prompt + each row's private pages) and their number rarely fits the
// SM count (8 sessions x 8 heads = 64 groups, 32 x 8 = 256 groups on 148
// SMs: 13% idle SMs / 1.73 waves). Here the groups' pages are laid end to end
// and cut into gridDim.x equal runs (one persistent CTA per SM): a run is a
// sequence of segments, one per group it touches. The producer streams the
// whole run through one TMA ring without a break; the consumer warps process
// it segment by segment (Q of the segment's group staged, the same
// mma.sync flash loop as decode_attn_partial, fold, one (m, l, o) partial
// per segment in slot cta + group, which is unique because successive
// segments advance the CTA, the group, or both). The CTA holding a group's
// first page records {first, last CTA} of the group for the merge kernel.
namespace sk {

// Consumers wait on `full` by parity: a warp must never wait for round r of
// a stage before round r - 1 of it completed (it could mistake round r - 2's
// parity), so NST is a multiple of every `ways` (8 / 4 / 2) and segments are
// separated by consumer barriers.
constexpr int NST = 16;                         // 128 KiB ring
constexpr int MAXS = 64;                        // sessions (tables in shared memory)
constexpr int MAXP = 2048;                      // pages of one run
constexpr int OFF_Q = NST * STAGE;
constexpr int OFF_SCR = OFF_Q;                  // fold scratch aliases Q (barrier-separated)
constexpr int OFF_BAR = OFF_SCR + CW * 32 * FRAG * 4;
constexpr int OFF_PG = OFF_BAR + 2 * NST * 8;
constexpr int SMEM = OFF_PG + MAXP * 4 + 1024;
static_assert(NST % CW == 0, "parity waits need NST % ways == 0");

struct Tables {
  int rows[MAXS][MAXR];
  int plen[MAXS][MAXR];
  int pstart[MAXS][MAXR + 1];  // page index (within the group) of each row's first private page
  int nsh[MAXS];               // shared pages
  int ls[MAXS];
  int nr[MAXS];
  int P[MAXS];                 // pages per group of the session (0 without rows)
  int off[MAXS + 1];           // prefix of P over sessions
};

__device__ __forceinline__ int run_begin(int c, int64_t total, int grid) { return (int)((int64_t)c * total / grid); }

// session / head / page of flat page index x (x < total)
__device__ __forceinline__ void locate(const Tables& t, int n_sess, int nkv, int x, int& s, int& h, int& k) {
  int lo = 0, hi = n_sess - 1;  // largest s with nkv * off[s] <= x
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (nkv * t.off[mid] <= x) lo = mid;
    else hi = mid - 1;
  }
  s = lo;
  const int r = x - nkv * t.off[s];
  h = r / t.P[s];
  k = r % t.P[s];
}

__device__ __forceinline__ int cta_of(int x, int64_t total, int grid) {
  int c = (int)((int64_t)x * grid / total);
  while (c + 1 < grid && run_begin(c + 1, total, grid) <= x) ++c;
  while (c > 0 && run_begin(c, total, grid) > x) --c;
  return c;
}

__device__ __forceinline__ void mbar_arrive_n(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0], %1;" ::"r"(tma::sa(bar)), "r"(n) : "memory");
}

__global__ void __launch_bounds__(THREADS, 1)
    decode_attn_sk(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t* empty = full + NST;
  int* s_page = reinterpret_cast<int*>(smem + OFF_PG);
  float* scr = reinterpret_cast<float*>(smem + OFF_SCR);  // [CW][32][FRAG]
  __shared__ Tables t;
  __shared__ int64_t s_total;

  trace_stamp(0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nkv = p.kv.n_kv_heads, nS = p.b.n_sess;
  const int grid = gridDim.x, cta = blockIdx.x;

  // ---- session tables: one thread per (session, row) pair, two load rounds
  for (int e = threadIdx.x; e < nS * MAXR; e += THREADS) {
    const int sx = e / MAXR, i = e % MAXR;
    const int nr = p.b.sess_nrows[sx];
    if (i < nr) {
      const int r = p.b.sess_rows[(int64_t)sx * p.b.max_rows_per_sess + i];
      t.rows[sx][i] = r;
      t.plen[sx][i] = p.b.priv_len[r] + 1;  // includes the token appended this step
    }
    if (i == 0) {
      t.nr[sx] = nr;
      t.ls[sx] = p.b.sess_len[sx];
    }
  }
  if (threadIdx.x == 0) {
    for (int st = 0; st < NST; ++st) {
      tma::mbar_init(&full[st], 1);
      tma::mbar_init(&empty[st], CW);
    }
    tma::fence_mbar_init();
    tma::prefetch_map(&kvmap);
  }
  __syncthreads();
  for (int sx = threadIdx.x; sx < nS; sx += THREADS) {
    const int nsh = (t.ls[sx] + PT - 1) / PT;
    int acc = nsh;
    for (int i = 0; i < t.nr[sx]; ++i) {
      t.pstart[sx][i] = acc;
      acc += (t.plen[sx][i] + PT - 1) / PT;
    }
    t.pstart[sx][t.nr[sx]] = acc;
    t.nsh[sx] = nsh;
    t.P[sx] = t.nr[sx] > 0 ? acc : 0;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int sx = 0; sx < nS; ++sx) {
      t.off[sx] = acc;
      acc += t.P[sx];
    }
    t.off[nS] = acc;
    s_total = (int64_t)acc * nkv;
  }
  __syncthreads();
  const int64_t total = s_total;
  // the merge needs the run boundaries too: CTAs with empty runs (fewer pages
  // than SMs) write no partial and are skipped
  if (cta == 0 && threadIdx.x == 0) p.dir[2 * nS * nkv] = (int)total;
  const int c0 = run_begin(cta, total, grid), c1 = run_begin(cta + 1, total, grid);
  const int np = c1 - c0;
  auto page_at = [&](int sx, int hh, int kk) -> int {
    (void)hh;
    if (kk < t.nsh[sx]) return p.b.sess_pages[(int64_t)sx * p.b.max_sess_pages + kk];
    int i = 0;
    while (kk >= t.pstart[sx][i + 1]) ++i;
    return p.b.row_pages[(int64_t)t.rows[sx][i] * p.b.max_row_pages + (kk - t.pstart[sx][i])];
  };
  // page ids of the run -> shared memory
  for (int j = threadIdx.x; j < np && j < MAXP; j += THREADS) {
    int sx, hh, kk;
    locate(t, nS, nkv, c0 + j, sx, hh, kk);
    s_page[j] = page_at(sx, hh, kk);
  }
  __syncthreads();
  trace_stamp(1);
  asm volatile("griddepcontrol.wait;" ::: "memory");  // q / the appended K,V come from rope_append

  if (warp == CW) {
    // ---------------- TMA producer: the whole run, one ring ----------------
    if (lane == 0 && np > 0) {
      int sx, hh, kk;
      locate(t, nS, nkv, c0, sx, hh, kk);
      for (int j = 0; j < np; ++j) {
        const int st = j % NST;
        tma::mbar_wait(&empty[st], ((j / NST) & 1) ^ 1);
        const int page = j < MAXP ? s_page[j] : page_at(sx, hh, kk);
        const int row_k = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv + hh) * PT);
        tma::mbar_expect_tx(&full[st], STAGE);
        tma::load_4d(&kvmap, &full[st], smem + st * STAGE, 0, row_k, 0, 0);
        if (++kk == t.P[sx]) {  // next group
          kk = 0;
          if (++hh == nkv) {
            hh = 0;
            do ++sx; while (sx < nS && t.P[sx] == 0);
          }
        }
      }
    }
    // lanes 1-31 must not exit while lane 0 issues TMA (the issue sequence
    // uses warp-uniform registers: exited lanes make it an illegal instruction)
    __syncwarp();
  } else if (np > 0) {
    // ---------------- consumers: segment by segment ----------------
    const uint32_t ring = smem_u32(smem);
    int sx, hh, kk;
    locate(t, nS, nkv, c0, sx, hh, kk);
    int c = c0, j0 = 0;
    while (c < c1) {
      const int n = min(t.P[sx] - kk, c1 - c);
      const int nr = t.nr[sx];
      const int G = nr * p.grp;
      const int T = (G + 15) / 16;
      const int Tp = T <= 1 ? 1 : (T == 2 ? 2 : 4);
      const int ways = CW / Tp;
      const int g = sx * nkv + hh;  // group
      // Q of this group -> shared (the previous segment is fully folded)
      {
        const uint32_t qs = smem_u32(smem + OFF_Q);
        for (int e = threadIdx.x; e < T * 16 * 16; e += CW * 32) {
          const int gq = e >> 4, cc = e & 15;
          uint4 v = make_uint4(0, 0, 0, 0);
          if (gq < G) {
            const int qh = hh * p.grp + gq % p.grp;
            v = *reinterpret_cast<const uint4*>(p.q + ((int64_t)t.rows[sx][gq / p.grp] * p.nq + qh) * HD + cc * 8);
          }
          asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(qs + swz256(gq, cc)), "r"(v.x),
                       "r"(v.y), "r"(v.z), "r"(v.w));
        }
      }
      named_barrier_sync(1, CW * 32);
      if (c == c0) trace_stamp(2);
      const int tile = warp / ways, way = warp % ways;
      const bool active = tile < T;
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
        for (int q = way; q < n; q += ways) {
          const int j = j0 + q;
          const int st = j % NST;
          // parity waits are safe: within a segment stage s is read by one
          // warp per m-tile in every round (NST % ways == 0), and a segment
          // starts only after every page of the previous one was consumed
          tma::mbar_wait(&full[st], (j / NST) & 1);
          const int kq = kk + q;
          int limit, owner;
          if (kq < t.nsh[sx]) {
            limit = min(PT, t.ls[sx] - kq * PT);
            owner = -1;
          } else {
            int i = 0;
            while (kq >= t.pstart[sx][i + 1]) ++i;
            limit = min(PT, t.plen[sx][i] - (kq - t.pstart[sx][i]) * PT);
            owner = i;
          }
          const uint32_t kt = ring + st * STAGE, vt = kt + TILE;
          float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
          {
            const int mi = lane >> 3, ri = lane & 7;
            const int tok = (mi >> 1) * 8 + ri;
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              uint32_t b0, b1, b2, b3;
              ldmatrix_x4(tile_addr(kt, tok, 2 * ks + (mi & 1)), b0, b1, b2, b3);
              mma_bf16_16816(sc[0], qa[ks], b0, b1);
              mma_bf16_16816(sc[1], qa[ks], b2, b3);
            }
          }
          const bool okA = owner < 0 || owner == ownA;
          const bool okB = owner < 0 || owner == ownB;
          const int cb = (lane & 3) * 2;
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const int tt = nt * 8 + cb + (e & 1);
              const bool ok = tt < limit && (e < 2 ? okA : okB);
              sc[nt][e] = ok ? sc[nt][e] * p.scale_log2 : -INFINITY;
            }
          float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
          float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
          const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
          const float r0 = n0 == -INFINITY ? 0.f : n0, r1 = n1 == -INFINITY ? 0.f : n1;
          const float c0f = fast_exp2(m0 - r0), c1f = fast_exp2(m1 - r1);
          m0 = n0;
          m1 = n1;
          float pr[2][4];
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) {
            pr[nt][0] = fast_exp2(sc[nt][0] - r0);
            pr[nt][1] = fast_exp2(sc[nt][1] - r0);
            pr[nt][2] = fast_exp2(sc[nt][2] - r1);
            pr[nt][3] = fast_exp2(sc[nt][3] - r1);
          }
          l0 = l0 * c0f + ((pr[0][0] + pr[0][1]) + (pr[1][0] + pr[1][1]));
          l1 = l1 * c1f + ((pr[0][2] + pr[0][3]) + (pr[1][2] + pr[1][3]));
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            o[i][0] *= c0f;
            o[i][1] *= c0f;
            o[i][2] *= c1f;
            o[i][3] *= c1f;
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
          // every stage gets CW arrivals: one per m-tile that read it, the
          // tile-0 warp adds the CW - T of the tiles this segment lacks
          if (lane == 0) mbar_arrive_n(&empty[st], tile == 0 ? (uint32_t)(CW - T + 1) : 1u);
        }
        l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
        l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
        l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
      }
      // ---- fold the `ways` warps of each m-tile (scratch aliases Q: every
      // warp has its Q fragments in registers past this barrier) ----
      named_barrier_sync(1, CW * 32);
      if (active) {
        float4* d = reinterpret_cast<float4*>(scr + (warp * 32 + lane) * FRAG);
#pragma unroll
        for (int i = 0; i < 16; ++i) d[i] = make_float4(o[i][0], o[i][1], o[i][2], o[i][3]);
        d[16] = make_float4(m0, m1, l0, l1);
      }
      named_barrier_sync(1, CW * 32);
      const int64_t base = (int64_t)(cta + g) * GMAX;
      {
        const int ra = lane >> 2, rb = ra + 8, cb = (lane & 3) * 2;
        for (int tt = 0; tt < T; ++tt) {
          float Ma = -INFINITY, Mb = -INFINITY;
          for (int v = 0; v < ways; ++v) {
            const float4 ml = reinterpret_cast<const float4*>(scr + ((tt * ways + v) * 32 + lane) * FRAG)[16];
            Ma = fmaxf(Ma, ml.x);
            Mb = fmaxf(Mb, ml.y);
          }
          const float Mra = Ma == -INFINITY ? 0.f : Ma, Mrb = Mb == -INFINITY ? 0.f : Mb;
          float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
          float La = 0.f, Lb = 0.f;
          for (int v = 0; v < ways; ++v) {
            const float* src = scr + ((tt * ways + v) * 32 + lane) * FRAG;
            const float4 ml = reinterpret_cast<const float4*>(src)[16];
            const float fa = exp2f(ml.x - Mra), fb = exp2f(ml.y - Mrb);
            La += fa * ml.z;
            Lb += fb * ml.w;
            const float4 x0 = reinterpret_cast<const float4*>(src)[2 * warp];
            const float4 x1 = reinterpret_cast<const float4*>(src)[2 * warp + 1];
            acc[0] += fa * x0.x; acc[1] += fa * x0.y; acc[2] += fb * x0.z; acc[3] += fb * x0.w;
            acc[4] += fa * x1.x; acc[5] += fa * x1.y; acc[6] += fb * x1.z; acc[7] += fb * x1.w;
          }
          const int ga = tt * 16 + ra, gb = tt * 16 + rb;
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
      if (kk == 0 && threadIdx.x == 0) {  // this run holds the group's first page
        const int x_last = nkv * t.off[sx] + hh * t.P[sx] + t.P[sx] - 1;
        p.dir[2 * g] = cta;
        p.dir[2 * g + 1] = cta_of(x_last, total, grid);
      }
      named_barrier_sync(1, CW * 32);  // scratch and Q are rewritten by the next segment
      // next segment
      c += n;
      j0 += n;
      kk += n;
      if (kk == t.P[sx]) {
        kk = 0;
        if (++hh == nkv) {
          hh = 0;
          do ++sx; while (sx < nS && t.P[sx] == 0);
        }
      }
    }
  }
  trace_stamp(3);
  asm volatile("griddepcontrol.launch_dependents;");
  trace_stamp(4);
}

}  // namespace sk


// ------------------------------------------- all-heads partial kernel (H) --
// The (session, split) CTA of this kernel owns ALL KV heads of its pages:
// one 4-D TMA box per page brings the page's whole K|V block of this layer
// (nkv heads x 16 tokens x 128 dims x K|V = 64 KiB at the 8B shape, one
// contiguous run) and consumer warp h runs the flash loop of KV head h over
// every page of the split. Versus decode_attn_partial (CTA = one head, 8 KiB
// boxes) this reads DRAM in 64 KiB runs, needs 8x fewer CTAs for the same
// work (agent serving: one session per row, 8 heads -> 2048 small CTAs
// become 256) and no cross-warp fold (each warp owns its head's softmax
// state). Used when every session has <= 16 query rows per KV head (one m16
// tile, e.g. 4 modules x 4 GQA heads); the partial format is the same as
// decode_attn_partial's, so decode_attn_merge is shared.
namespace hk {

constexpr int NST = 3;
constexpr int MAXKV = 8;                       // consumer warps = KV heads
__host__ __device__ constexpr int stage_bytes(int nkv) { return 2 * nkv * TILE; }  // K|V x heads x 4 KiB
constexpr int STAGE_MAX = stage_bytes(MAXKV);   // 64 KiB
constexpr int OFF_Q = 2 * STAGE_MAX;            // Q is staged in ring stage 2 before the stream starts
constexpr int OFF_BAR = NST * STAGE_MAX;         // 192 KiB
constexpr int OFF_PG = OFF_BAR + 2 * NST * 8;
constexpr int SMEM = OFF_PG + 1024 * 4 + 1024;  // (page ids of up to 1024 pages staged)
constexpr int MAXP_SMEM = 1024;
constexpr int THREADS = (MAXKV + 1) * 32;

__global__ void __launch_bounds__(THREADS, 1)
    decode_attn_heads(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ Params p) {
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
  const int sess = item / p.ns;
  const int nr = p.b.sess_nrows[sess];
  const int G = nr * p.grp;  // query rows per KV head (<= 16)
  const int STG = stage_bytes(nkv);

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
    s_total = nr > 0 ? acc : 0;
    for (int st = 0; st < NST; ++st) {
      tma::mbar_init(&full[st], 1);
      tma::mbar_init(&empty[st], nkv);
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
  for (int j = threadIdx.x; j < np && j < MAXP_SMEM; j += THREADS) s_page[j] = page_of(k0 + j);
  // The producer streams the first two ring stages of shared prompt pages
  // before the PDL wait (no kernel of a decode step writes them; see
  // psk_decode_attn); stage 2 holds Q until the stream starts.
  int pre = 0;
  if (p.early && threadIdx.x == MAXKV * 32) {
    for (; pre < NST - 1 && pre < np && k0 + pre < s_ps; ++pre) {
      const int page = page_of(k0 + pre);
      const int row0 = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv) * PT);
      tma::mbar_expect_tx(&full[pre], STG);
      tma::load_4d(&kvmap, &full[pre], smem + pre * STAGE_MAX, 0, row0, 0, 0);
    }
  }
  asm volatile("griddepcontrol.wait;" ::: "memory");  // q / the appended K,V come from rope_append
  // Q of every head: rows g of head h at [h][16][256 B] (swizzled)
  {
    // all loads in flight first (one latency round trip), then the stores
    constexpr int QPER = (MAXKV * 16 * 16 + THREADS - 1) / THREADS;
    const uint32_t qs = smem_u32(smem + OFF_Q);
    uint4 v[QPER];
#pragma unroll
    for (int u = 0; u < QPER; ++u) {
      const int e = threadIdx.x + u * THREADS;
      const int hh = e >> 8, g = (e >> 4) & 15, c = e & 15;
      v[u] = make_uint4(0, 0, 0, 0);
      if (hh < nkv && g < G)
        v[u] = __ldg(reinterpret_cast<const uint4*>(p.q + ((int64_t)s_rows[g / p.grp] * p.nq + hh * p.grp + g % p.grp) *
                                                               HD + c * 8));
    }
#pragma unroll
    for (int u = 0; u < QPER; ++u) {
      const int e = threadIdx.x + u * THREADS;
      const int hh = e >> 8, g = (e >> 4) & 15, c = e & 15;
      if (hh < nkv)
        asm volatile("st.shared.v4.u32 [%0], {%1,%2,%3,%4};" ::"r"(qs + hh * 4096 + swz256(g, c)), "r"(v[u].x),
                     "r"(v[u].y), "r"(v[u].z), "r"(v[u].w));
    }
  }
  __syncthreads();
  // Q fragments -> registers before the producer may overwrite stage 2
  uint32_t qa[8][4];
  if (warp < nkv) {
    const uint32_t qs = smem_u32(smem + OFF_Q) + warp * 4096;
    const int qrow = ((lane >> 3) & 1) * 8 + (lane & 7);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks)
      ldmatrix_x4(qs + swz256(qrow, 2 * ks + (lane >> 4)), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
  }
  __syncthreads();
  trace_stamp(2);

  if (warp == MAXKV) {
    // ---------------- TMA producer: one box per page, all heads ----------------
    if (lane == 0) {
      for (int j = pre; j < np; ++j) {
        const int st = j % NST;
        tma::mbar_wait(&empty[st], ((j / NST) & 1) ^ 1);
        const int page = j < MAXP_SMEM ? s_page[j] : page_of(k0 + j);
        const int row0 = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv) * PT);
        tma::mbar_expect_tx(&full[st], STG);
        tma::load_4d(&kvmap, &full[st], smem + st * STAGE_MAX, 0, row0, 0, 0);
      }
    }
    __syncwarp();
  } else if (warp < nkv) {
    const int h = warp;
    const uint32_t ring = smem_u32(smem);
    const int half_stride = nkv * PT * 128;  // bytes between the dims 0-63 and 64-127 boxes
    float o[16][4];
#pragma unroll
    for (int i = 0; i < 16; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    const int gA = lane >> 2, gB = gA + 8;
    const int ownA = gA < G ? gA / p.grp : -2, ownB = gB < G ? gB / p.grp : -2;
    for (int j = 0; j < np; ++j) {
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
      // head h: K rows [16h, 16h+16) of the box, V nkv*16 rows later
      const uint32_t kt = ring + st * STAGE_MAX + h * (PT * 128);
      const uint32_t vt = kt + 2 * half_stride;
      float sc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
      {
        const int mi = lane >> 3, ri = lane & 7;
        const int tok = (mi >> 1) * 8 + ri;
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          const int c16 = 2 * ks + (mi & 1);
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4(kt + (c16 >> 3) * half_stride + tok * 128 + (((c16 & 7) ^ (tok & 7)) << 4), b0, b1, b2, b3);
          mma_bf16_16816(sc[0], qa[ks], b0, b1);
          mma_bf16_16816(sc[1], qa[ks], b2, b3);
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
          sc[nt][e] = ok ? sc[nt][e] * p.scale_log2 : -INFINITY;
        }
      float mx0 = fmaxf(fmaxf(sc[0][0], sc[0][1]), fmaxf(sc[1][0], sc[1][1]));
      float mx1 = fmaxf(fmaxf(sc[0][2], sc[0][3]), fmaxf(sc[1][2], sc[1][3]));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float n0 = fmaxf(m0, mx0), n1 = fmaxf(m1, mx1);
      const float r0 = n0 == -INFINITY ? 0.f : n0, r1 = n1 == -INFINITY ? 0.f : n1;
      const float c0f = fast_exp2(m0 - r0), c1f = fast_exp2(m1 - r1);
      m0 = n0;
      m1 = n1;
      float pr[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        pr[nt][0] = fast_exp2(sc[nt][0] - r0);
        pr[nt][1] = fast_exp2(sc[nt][1] - r0);
        pr[nt][2] = fast_exp2(sc[nt][2] - r1);
        pr[nt][3] = fast_exp2(sc[nt][3] - r1);
      }
      l0 = l0 * c0f + ((pr[0][0] + pr[0][1]) + (pr[1][0] + pr[1][1]));
      l1 = l1 * c1f + ((pr[0][2] + pr[0][3]) + (pr[1][2] + pr[1][3]));
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        o[i][0] *= c0f;
        o[i][1] *= c0f;
        o[i][2] *= c1f;
        o[i][3] *= c1f;
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
          const int c16 = 2 * np2 + (mi >> 1);
          uint32_t b0, b1, b2, b3;
          ldmatrix_x4_trans(vt + (c16 >> 3) * half_stride + tok * 128 + (((c16 & 7) ^ (tok & 7)) << 4), b0, b1,
                            b2, b3);
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
    // partial (m, l, o) of head h's rows: same slots as decode_attn_partial
    const int64_t base = ((int64_t)(sess * nkv + h) * p.ns + j_split) * GMAX;
    const int cb = (lane & 3) * 2;
#pragma unroll
    for (int nt = 0; nt < 16; ++nt) {
      const int col = nt * 8 + cb;
      if (gA < G) *reinterpret_cast<float2*>(p.po + (base + gA) * HD + col) = make_float2(o[nt][0], o[nt][1]);
      if (gB < G) *reinterpret_cast<float2*>(p.po + (base + gB) * HD + col) = make_float2(o[nt][2], o[nt][3]);
    }
    if ((lane & 3) == 0) {
      if (gA < G) {
        p.pm[base + gA] = m0;
        p.pl[base + gA] = l0;
      }
      if (gB < G) {
        p.pm[base + gB] = m1;
        p.pl[base + gB] = l1;
      }
    }
  }
  trace_stamp(3);
  if (!p.fused) {
    asm volatile("griddepcontrol.launch_dependents;");
    return;
  }
  // In-kernel merge (the session's splits are co-resident): wait for them,
  // then fold slice j_split of the session's (head, row, 4 dims) outputs.
  split_barrier(p.cnt + 2 * sess * nkv, (unsigned)p.ns);
  __syncthreads();
  trace_stamp(4);
  const int GT = G * (HD / 4), T = nkv * GT;
  const int t0 = (int)((int64_t)j_split * T / p.ns), t1 = (int)((int64_t)(j_split + 1) * T / p.ns);
  for (int t = t0 + (int)threadIdx.x; t < t1; t += THREADS) {
    const int h = t / GT, rem = t - h * GT;
    const int g = rem >> 5, d4 = (rem & 31) * 4;
    const int64_t base = (int64_t)(sess * nkv + h) * p.ns * GMAX + g;
    float M = -INFINITY;
    for (int s = 0; s < p.ns; ++s) M = fmaxf(M, __ldcg(p.pm + base + (int64_t)s * GMAX));
    const float Mr = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 4
    for (int s = 0; s < p.ns; ++s) {
      const int64_t sl = base + (int64_t)s * GMAX;
      const float f = exp2f(__ldcg(p.pm + sl) - Mr);
      const float4 o = __ldcg(reinterpret_cast<const float4*>(p.po + sl * HD + d4));
      L += f * __ldcg(p.pl + sl);
      acc.x += f * o.x;
      acc.y += f * o.y;
      acc.z += f * o.z;
      acc.w += f * o.w;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
        p.out + ((int64_t)s_rows[g / p.grp] * p.nq + h * p.grp + g % p.grp) * HD + d4);
    dst[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    dst[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  }
}

}  // namespace hk

// Merge: one CTA per (row, q head), one thread per head dim; every split's
// (m, l, o) is loaded up front (32 splits in flight per thread) and folded by
// log-sum-exp. Launched with programmatic dependent launch: it is scheduled
// while the partial kernel drains and waits on griddepcontrol for its data.
constexpr int MERGE_U = 8;  // partials in flight per iteration (32 held 124 registers: 4 CTAs/SM)
__global__ void __launch_bounds__(HD) decode_attn_merge(const __grid_constant__ Params p) {
  const int r = blockIdx.x, qh = blockIdx.y, d = threadIdx.x;
  const int nkv = p.kv.n_kv_heads;
  const int h = qh / p.grp;
  // the row tables are static within a step: read them before the wait
  const int g = p.b.row_in_sess[r] * p.grp + qh % p.grp;
  const int grp_id = p.b.row_sess[r] * nkv + h;
  // let the next kernel (the o-proj GEMV streaming its weights) be scheduled
  // now: its own griddepcontrol.wait still waits for this grid to complete
  asm volatile("griddepcontrol.launch_dependents;");
  asm volatile("griddepcontrol.wait;" ::: "memory");
  // partial slots of this (session, KV head): splits mode ns consecutive
  // slots; stream-K mode slots cta + group for the CTAs in dir[group]
  int64_t first;
  int n, cf = 0;
  int64_t total = 0;
  if (p.ns > 0) {
    first = (int64_t)grp_id * p.ns;
    n = p.ns;
  } else {
    cf = p.dir[2 * grp_id];
    const int cl = p.dir[2 * grp_id + 1];
    total = p.dir[2 * p.b.n_sess * nkv];
    first = (int64_t)cf + grp_id;
    n = cl - cf + 1;
  }
  const int64_t base = first * GMAX + g;
  float M = -INFINITY, L = 0.f, acc = 0.f;
  for (int j0 = 0; j0 < n; j0 += MERGE_U) {
    float mj[MERGE_U], lj[MERGE_U], oj[MERGE_U];
#pragma unroll
    for (int u = 0; u < MERGE_U; ++u) {
      const int j = j0 + u;
      const int64_t sl = base + (int64_t)j * GMAX;
      bool ok = j < n;
      if (ok && p.ns == 0 && total < p.sk_grid) {  // stream-K, fewer pages than CTAs: skip empty runs
        const int c = cf + j;
        ok = sk::run_begin(c, total, p.sk_grid) != sk::run_begin(c + 1, total, p.sk_grid);
      }
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
// 5th-gen tensor cores with the same CTA = (session, kv head, split) work
// split and the same (m, l, o) partial format, so the merge kernel is shared.
//   warp 0     TMA producer (warp-converged, one elected lane issues): 4
//              pages per 64-key chunk, 6 stages; each page as ONE 4-D box,
//              its K and V for this (layer, head): [K|V][dims 0-63 |
//              64-127][16][64], 8 KiB, 128B-swizzled, pages 8 KiB apart
//   warp 1     MMA issuer (warp-converged) + TMEM owner. Q and P live in TMEM (A operand
//              from tensor memory): S_u = Q K^T as two M128 N32 MMAs per
//              16-dim K-step whose B rows are the SW128 atoms of the 4 pages
//              at an 8 KiB stride (tokens 0-7 of pages 0-3, then tokens
//              8-15), and O_u += P_u V_p (M128 N128 K16, one per page)
//   warps 2-9  two softmax groups u = 0, 1 taking alternate chunks, with
//              separate TMEM accumulators O_0, O_1 and separate (m, l): the
//              tensor core runs one group's MMAs while the other group does
//              its softmax; O is rescaled in TMEM only when a row max grows
//              by > 2^8 (lazy, exact after the final 1/l). At the end group 0
//              folds O_1 into O_0 and writes the split partial; when the
//              grid is one wave the split CTAs then merge their group
//              themselves (fused_merge), otherwise decode_attn_merge runs.
// Query rows = TMEM lanes (rows >= G are never read), so only the warps
// whose lane quarter holds live rows take part in the softmax.
// TMEM columns: S_0 [0,64) S_1 [64,128) O_0 [128,256) O_1 [256,384)
//               Q [384,448) (bf16 pairs) P_0 [448,480) P_1 [480,512).
// S column 32 hh + 8 pp + t holds token 8 hh + t of page pp; P is stored in
// page order (the PV MMA's K order), a register permutation.
// (TMA ops cost ~60-80 ns each whatever their size below ~4 KiB, so ops
// per page bound the stream: the earlier layout, K as two [16 x 64] 2-D
// boxes + V as one 3-D box per page so one N=64 MMA covered the chunk, took
// 3 ops per page; per-page N=16 S MMAs cost more in MMA issue: 54 vs 39 us at
// 32k x 16 modules.)
namespace tcv {

constexpr int CPG = 4;                  // pages per chunk
constexpr int KC = CPG * PT;            // 64 keys
#ifndef PSK_FANOUT_NSTG
#define PSK_FANOUT_NSTG 6  // ring stages (32 KiB each)
#endif
constexpr int NSTG = PSK_FANOUT_NSTG;
constexpr int PGB = 2 * TILE;           // 8 KiB per page: [K|V][half][16][64]
constexpr int STG = CPG * PGB;          // 32 KiB per chunk
constexpr int OFF_ML = NSTG * STG;
constexpr int OFF_BAR = OFF_ML + 128 * 8;
constexpr int OFF_PG = OFF_BAR + 256;
constexpr int OFF_INFO = OFF_PG + MAXP * 4;
constexpr int SMEM = OFF_INFO + MAXP * 4 + 1024;
constexpr int THREADS = 320;
constexpr uint32_t T_S = 0, T_O = 128, T_Q = 384, T_P = 448;
constexpr float RESCALE_LOG2 = 8.f;

// Slice j of a (session, KV head) group's split merge: the group's (query
// row, 4 dims) outputs [j T / ns, (j + 1) T / ns), each folded over the ns
// split partials by log-sum-exp. (Measured and kept over K lanes per output
// with all partials' loads in flight + shuffle combine: no faster at 32k x 16
// modules, slower at 8 sessions x 4k; tools/k6_ab.py.)
template <int NT>
__device__ __forceinline__ void merge_slice(const Params& p, int grp_id, int j, int h, int G, const int* rows) {
  const int T = G * (HD / 4);
  const int t0 = (int)((int64_t)j * T / p.ns), t1 = (int)((int64_t)(j + 1) * T / p.ns);
  for (int t = t0 + (int)threadIdx.x; t < t1; t += NT) {
    const int g = t >> 5, d4 = (t & 31) * 4;
    const int64_t base = (int64_t)grp_id * p.ns * GMAX + g;
    float M = -INFINITY;
#pragma unroll 8
    for (int s = 0; s < p.ns; ++s) M = fmaxf(M, __ldcg(p.pm + base + (int64_t)s * GMAX));
    const float Mr = M == -INFINITY ? 0.f : M;
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 6
    for (int s = 0; s < p.ns; ++s) {
      const int64_t sl = base + (int64_t)s * GMAX;
      const float f = exp2f(__ldcg(p.pm + sl) - Mr);
      const float4 o = __ldcg(reinterpret_cast<const float4*>(p.po + sl * HD + d4));
      L += f * __ldcg(p.pl + sl);
      acc.x += f * o.x;
      acc.y += f * o.y;
      acc.z += f * o.z;
      acc.w += f * o.w;
    }
    const float inv = L > 0.f ? 1.f / L : 0.f;
    const int qh = h * p.grp + g % p.grp;
    __nv_bfloat162* dst = reinterpret_cast<__nv_bfloat162*>(
        p.out + ((int64_t)rows[g / p.grp] * p.nq + qh) * HD + d4);
    dst[0] = __floats2bfloat162_rn(acc.x * inv, acc.y * inv);
    dst[1] = __floats2bfloat162_rn(acc.z * inv, acc.w * inv);
  }
}

// Fused merge of the fan-out kernel: after publishing its partial each
// split CTA waits for the group's other splits (split_barrier) and merges a
// 1/ns slice of the group's (query row, 4 dims) outputs by log-sum-exp,
// instead of a second kernel that waits for the whole grid.
__device__ __forceinline__ void fused_merge(const Params& p, int grp_id, int j, int h, int G, const int* s_rows) {
  split_barrier(p.cnt + 2 * grp_id, (unsigned)p.ns);
  ring_stamp(p, 5);
  __syncthreads();
  merge_slice<THREADS>(p, grp_id, j, h, G, s_rows);
}

__global__ void __launch_bounds__(THREADS, 1)
    decode_attn_tc(const __grid_constant__ CUtensorMap kvmap, const __grid_constant__ Params p) {
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
  uint64_t *full = bars, *empty = bars + NSTG, *s_full = bars + 2 * NSTG, *p_full = s_full + 2,
           *pv_done = p_full + 2, *g1_done = pv_done + 2, *s_free = g1_done + 1;
  int* s_page = reinterpret_cast<int*>(smem + OFF_PG);
  int* s_info = reinterpret_cast<int*>(smem + OFF_INFO);  // (owner + 1) << 8 | valid tokens
  float* s_ml = reinterpret_cast<float*>(smem + OFF_ML);  // group 1 (m, l) per row
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
  // Query row g sits in TMEM lane 32 * (g / 16) + g % 16: 16 live lanes per
  // lane quarter, so all four SM sub-partitions run softmax warps.
  const int act = (G + 15) / 16;  // softmax warps with live rows, per group

  trace_stamp(0);
  ring_stamp(p, 0);
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
    for (int s = 0; s < NSTG; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], 1);
    }
    for (int u = 0; u < 2; ++u) {
      tma::mbar_init(&s_full[u], 1);
      tma::mbar_init(&s_free[u], 32 * act);
      tma::mbar_init(&p_full[u], 32 * act);
      tma::mbar_init(&pv_done[u], 1);
    }
    tma::mbar_init(g1_done, 32 * act);
    tma::fence_mbar_init();
    tma::prefetch_map(&kvmap);
  }
  if (warp == 1) umma::tmem_alloc(&s_tmem, 512);
  __syncthreads();
  trace_stamp(1);
  ring_stamp(p, 1);
  const int total = s_total;
  const int k0 = (int)((int64_t)j_split * total / p.ns);
  const int k1 = (int)((int64_t)(j_split + 1) * total / p.ns);
  const int np = k1 - k0;
  const int nch = (np + CPG - 1) / CPG;
  // page id and (owner row, valid tokens) of the split's j-th page
  auto page_of = [&](int j, int& info) -> int {
    const int k = k0 + j;
    if (k < s_ps) {
      info = min(PT, s_ls - k * PT);
      return p.b.sess_pages[(int64_t)sess * p.b.max_sess_pages + k];
    }
    int i = 0;
    while (k >= s_pstart[i + 1]) ++i;
    info = ((i + 1) << 8) | min(PT, s_plen[i] - (k - s_pstart[i]) * PT);
    return p.b.row_pages[(int64_t)s_rows[i] * p.b.max_row_pages + (k - s_pstart[i])];
  };
  for (int j = threadIdx.x; j < np && j < MAXP; j += THREADS) {
    int info;
    s_page[j] = page_of(j, info);
    s_info[j] = info;
  }
  __syncthreads();
  const uint32_t tmem = s_tmem;
  // The producer (warp 0) streams the shared prompt pages at once (no kernel
  // of a decode step writes them); q and the private pages (this step's
  // appended token) come from rope_append, so everyone else waits (PDL).
  if (warp != 0) asm volatile("griddepcontrol.wait;" ::: "memory");
  // Q rows -> TMEM (lane = row, bf16 pairs), by the group-0 warps of live lanes
  if (warp >= 2 && warp < 6 && (warp & 3) < act) {
    const int g = lane < 16 ? (warp & 3) * 16 + lane : G;
    const uint32_t tq = tmem + ((uint32_t)((warp & 3) * 32) << 16) + T_Q;
    const uint4* src = nullptr;
    if (g < G)
      src = reinterpret_cast<const uint4*>(p.q + ((int64_t)s_rows[g / p.grp] * p.nq + h * p.grp + g % p.grp) * HD);
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      uint32_t r[32];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint4 v = src ? src[half * 8 + i] : make_uint4(0, 0, 0, 0);
        r[4 * i] = v.x;
        r[4 * i + 1] = v.y;
        r[4 * i + 2] = v.z;
        r[4 * i + 3] = v.w;
      }
      umma::st32(tq + half * 32, r);
    }
    umma::wait_st();
  }
  if (warp != 0) {
    umma::fence_before();
    named_barrier_sync(1, THREADS - 32);  // Q in TMEM (all but the producer)
    umma::fence_after();
  }
  trace_stamp(2);

  if (warp == 0) {
    // whole warp, warp-uniform operands, one elected lane issues (no
    // per-instruction waterfall loops)
    bool dep = false;
    for (int c = 0; c < nch; ++c) {
      const int st = c % NSTG;
      tma::mbar_wait(&empty[st], ((c / NSTG) & 1) ^ 1);
      // this step's private pages (and q) come from rope_append; the shared
      // prompt pages are written by no kernel of the step, so with p.early
      // they stream before the PDL wait
      if (!dep && (!p.early || k0 + c * CPG + CPG > s_ps)) {
        asm volatile("griddepcontrol.wait;" ::: "memory");
        dep = true;
      }
      tma::mbar_expect_tx_e(&full[st], STG);
#pragma unroll
      for (int pp = 0; pp < CPG; ++pp) {
        const int j = c * CPG + pp;
        const int jj = j < np ? j : 0;  // past the end: any valid page, masked
        int info;
        const int page = jj < MAXP ? s_page[jj] : page_of(jj, info);
        const int row_k = (int)((((int64_t)page * p.kv.n_layers + p.layer) * 2 * nkv + h) * PT);
        tma::load_4d_e(&kvmap, &full[st], smem + st * STG + pp * PGB, 0, row_k, 0, 0);  // K and V, 8 KiB
      }
      if (c == 0) ring_stamp(p, 2);
    }
    trace_stamp(3);
    ring_stamp(p, 3);
  } else if (warp == 1) {
    constexpr uint32_t ID_S = umma::idesc_bf16(128, KC / 2, false), ID_PV = umma::idesc_bf16(128, HD, true);
    auto issue_s = [&](int c) {
      const int u = c & 1;
      const uint32_t kb = smem_u32(smem + (c % NSTG) * STG);
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)  // tokens 8 hh .. 8 hh + 7 of the 4 pages
          umma::mma_ts_e(tmem + T_S + u * KC + hh * (KC / 2), tmem + T_Q + kk * 8,
                         umma::desc_k_sw128_sbo(kb + (kk >> 2) * 2048 + hh * 1024, PGB) + 2 * (kk & 3), ID_S,
                         kk > 0);
      umma::commit_e(&s_full[u]);
    };
    auto issue_pv = [&](int c) {
      const int u = c & 1;
      const uint32_t vb = smem_u32(smem + (c % NSTG) * STG) + TILE;
#pragma unroll
      for (int pp = 0; pp < CPG; ++pp)
        umma::mma_ts_e(tmem + T_O + u * HD, tmem + T_P + u * 32 + pp * 8, umma::desc_mn_sw128(vb + pp * PGB, 2048),
                       ID_PV, (c >= 2 || pp > 0) ? 1u : 0u);
      umma::commit_e(&pv_done[u]);
      umma::commit_e(&empty[c % NSTG]);
    };
    if (p.stream_only) {
      for (int c = 0; c < nch; ++c) {
        tma::mbar_wait(&full[c % NSTG], (c / NSTG) & 1);
        if (lane == 0) tma::mbar_arrive(&empty[c % NSTG]);
        __syncwarp();
      }
    }
    for (int c = 0; c < nch && c < 2 && !p.stream_only; ++c) {
      tma::mbar_wait(&full[c], 0);
      umma::fence_after();
      issue_s(c);
    }
    for (int c = 0; c < nch && !p.stream_only; ++c) {
      // S_u(c+2) as soon as softmax(c) has S_u(c) in registers, so it runs
      // under that softmax; then PV_u(c) once P_u(c) is in TMEM
      if (c + 2 < nch) {
        tma::mbar_wait(&s_free[c & 1], (c >> 1) & 1);
        tma::mbar_wait(&full[(c + 2) % NSTG], ((c + 2) / NSTG) & 1);
        umma::fence_after();
        issue_s(c + 2);
      }
      tma::mbar_wait(&p_full[c & 1], (c >> 1) & 1);  // P_u(c) in TMEM, O_u settled
      umma::fence_after();
      issue_pv(c);
    }
  } else if ((warp & 3) < act) {
    // Softmax warp: TMEM lane quarter q4, its 16 live lanes read with the
    // 16-lane shapes so all 32 threads work: thread t owns query rows
    // gA = 16 q4 + t/4 and gB = gA + 8, S columns 8i + 2(t%4) + {0,1}
    // (i = 0..7) = tokens 8 (i / 4) + 2(t%4) + {0,1} of page i % 4; the 4
    // threads of a row reduce with two shuffles.
    const int u = (warp - 2) >> 2;  // softmax group
    const int q4 = warp & 3;        // TMEM lane quarter
    const int t0 = lane & 3;
    const int gA = 16 * q4 + (lane >> 2), gB = gA + 8;
    const int riA = gA < G ? gA / p.grp : -2, riB = gB < G ? gB / p.grp : -2;
    const uint32_t tl = tmem + ((uint32_t)(32 * q4) << 16);
    const uint32_t tS = tl + T_S + u * KC, tO = tl + T_O + u * HD, tP = tl + T_P + u * 32;
    const float sc = p.scale_log2;
    float mA = -INFINITY, mB = -INFINITY, lA = 0.f, lB = 0.f;  // m in scaled log2 units
    int it = 0;
    for (int c = u; c < nch && !p.stream_only; c += 2, ++it) {
      tma::mbar_wait(&s_full[u], it & 1);
      umma::fence_after();
      uint32_t sr[32];
      umma::ld16x256b_x8(tS, sr);
      umma::wait_ld();
      umma::fence_before();
      tma::mbar_arrive(&s_free[u]);  // S_u may be overwritten by S_u(c+2)
      float xa[16], xb[16];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        xa[2 * i] = __uint_as_float(sr[4 * i]);
        xa[2 * i + 1] = __uint_as_float(sr[4 * i + 1]);
        xb[2 * i] = __uint_as_float(sr[4 * i + 2]);
        xb[2 * i + 1] = __uint_as_float(sr[4 * i + 3]);
      }
      int info[CPG];
      bool full = true;
#pragma unroll
      for (int pp = 0; pp < CPG; ++pp) {
        const int j = c * CPG + pp;
        info[pp] = 0;
        if (j < np) {
          if (j < MAXP) info[pp] = s_info[j];
          else page_of(j, info[pp]);
        }
        full = full && info[pp] == PT;  // whole shared page
      }
      if (!full) {  // warp-uniform: partial / private / past-the-end pages
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int inf = info[i & 3];
          const int own = (inf >> 8) - 1, lim = inf & 0xff;
          const bool okA = own < 0 || own == riA, okB = own < 0 || own == riB;
#pragma unroll
          for (int b = 0; b < 2; ++b) {
            const int e = 8 * (i >> 2) + 2 * t0 + b;
            if (!(okA && e < lim)) xa[2 * i + b] = -INFINITY;
            if (!(okB && e < lim)) xb[2 * i + b] = -INFINITY;
          }
        }
      }
      if (riA < 0) {
#pragma unroll
        for (int k = 0; k < 16; ++k) xa[k] = -INFINITY;
      }
      if (riB < 0) {
#pragma unroll
        for (int k = 0; k < 16; ++k) xb[k] = -INFINITY;
      }
      // tree max over the thread's 16 keys, then over the row's 4 threads
      float ta[8], tb[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        ta[k] = fmaxf(xa[2 * k], xa[2 * k + 1]);
        tb[k] = fmaxf(xb[2 * k], xb[2 * k + 1]);
      }
#pragma unroll
      for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) {
          ta[k] = fmaxf(ta[k], ta[k + w]);
          tb[k] = fmaxf(tb[k], tb[k + w]);
        }
      float mxA = ta[0], mxB = tb[0];
      mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 1));
      mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 1));
      mxA = fmaxf(mxA, __shfl_xor_sync(0xffffffffu, mxA, 2));
      mxB = fmaxf(mxB, __shfl_xor_sync(0xffffffffu, mxB, 2));
      mxA *= sc;
      mxB *= sc;
      if (it > 0) tma::mbar_wait(&pv_done[u], (it - 1) & 1);  // P_u free, O_u settled
      const bool growA = mxA > mA + RESCALE_LOG2 || (mA == -INFINITY && mxA > -INFINITY);
      const bool growB = mxB > mB + RESCALE_LOG2 || (mB == -INFINITY && mxB > -INFINITY);
      if (__any_sync(0xffffffffu, (growA || growB) && it > 0)) {
        umma::fence_after();
        const float alA = growA ? exp2f(mA - mxA) : 1.f, alB = growB ? exp2f(mB - mxB) : 1.f;
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          uint32_t o[32];
          umma::ld16x256b_x8(tO + hh * 64, o);
          umma::wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            o[4 * i] = __float_as_uint(__uint_as_float(o[4 * i]) * alA);
            o[4 * i + 1] = __float_as_uint(__uint_as_float(o[4 * i + 1]) * alA);
            o[4 * i + 2] = __float_as_uint(__uint_as_float(o[4 * i + 2]) * alB);
            o[4 * i + 3] = __float_as_uint(__uint_as_float(o[4 * i + 3]) * alB);
          }
          umma::st16x256b_x8(tO + hh * 64, o);
        }
        lA *= alA;
        lB *= alB;
      }
      if (growA) mA = mxA;
      if (growB) mB = mxB;
      const float bA = mA == -INFINITY ? 0.f : mA, bB = mB == -INFINITY ? 0.f : mB;
      // p = 2^(s * scale - m): masked keys are -inf -> 0
      uint32_t pk[16];
      float sa[8], sb[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        // P pair column 4i + t0 = tokens 8 (i & 1) + 2 t0 + {0,1} of page i / 2 = S group 4 (i & 1) + i / 2
        const int k = 4 * (i & 1) + (i >> 1);
        const float a0 = fast_exp2(fmaf(xa[2 * k], sc, -bA)), a1 = fast_exp2(fmaf(xa[2 * k + 1], sc, -bA));
        const float b0 = fast_exp2(fmaf(xb[2 * k], sc, -bB)), b1 = fast_exp2(fmaf(xb[2 * k + 1], sc, -bB));
        sa[i] = a0 + a1;
        sb[i] = b0 + b1;
        pk[2 * i] = pack_bf16(a0, a1);      // row A
        pk[2 * i + 1] = pack_bf16(b0, b1);  // row B
      }
      umma::st16x128b_x8(tP, pk);
#pragma unroll
      for (int w = 4; w >= 1; w >>= 1)
#pragma unroll
        for (int k = 0; k < w; ++k) {
          sa[k] += sa[k + w];
          sb[k] += sb[k + w];
        }
      lA += sa[0];
      lB += sb[0];
      umma::wait_st();
      umma::fence_before();
      tma::mbar_arrive(&p_full[u]);
    }
    if (it > 0) tma::mbar_wait(&pv_done[u], (it - 1) & 1);  // this group's last PV landed
    umma::fence_after();
    lA += __shfl_xor_sync(0xffffffffu, lA, 1);
    lB += __shfl_xor_sync(0xffffffffu, lB, 1);
    lA += __shfl_xor_sync(0xffffffffu, lA, 2);
    lB += __shfl_xor_sync(0xffffffffu, lB, 2);
    if (u == 1) {
      if (t0 == 0) {
        s_ml[2 * gA] = mA;
        s_ml[2 * gA + 1] = lA;
        s_ml[2 * gB] = mB;
        s_ml[2 * gB + 1] = lB;
      }
      umma::fence_before();
      tma::mbar_arrive(g1_done);
    } else {
      tma::mbar_wait(g1_done, 0);
      umma::fence_after();
      const bool has1 = nch > 1;  // group 1 ran at least one chunk (O_1 written)
      float a0[2], a1[2];
      const float m0r[2] = {mA, mB}, l0r[2] = {lA, lB};
      float Mr[2], Lr[2];
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const int g = r ? gB : gA;
        const float m1 = s_ml[2 * g], l1 = s_ml[2 * g + 1];
        const float M = fmaxf(m0r[r], m1);
        const float Mx = M == -INFINITY ? 0.f : M;
        a0[r] = m0r[r] == -INFINITY ? 0.f : exp2f(m0r[r] - Mx);
        a1[r] = (has1 && m1 != -INFINITY) ? exp2f(m1 - Mx) : 0.f;
        Mr[r] = M;
        Lr[r] = l0r[r] * a0[r] + (has1 ? l1 * a1[r] : 0.f);
      }
      const int64_t base = (int64_t)item * GMAX;
#pragma unroll 1
      for (int hh = 0; hh < 2; ++hh) {
        uint32_t o0[32], o1[32];
        umma::ld16x256b_x8(tO + hh * 64, o0);
        umma::ld16x256b_x8(tO + HD + hh * 64, o1);  // O_1 sits HD columns after O_0
        umma::wait_ld();
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const int g = r ? gB : gA;
          if (g >= G) continue;
          float* dst = p.po + (base + g) * HD + hh * 64 + 2 * t0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            float f[2];
#pragma unroll
            for (int e = 0; e < 2; ++e) {
              const int k = 4 * i + 2 * r + e;
              const float x0 = a0[r] != 0.f ? a0[r] * __uint_as_float(o0[k]) : 0.f;
              const float x1 = a1[r] != 0.f ? a1[r] * __uint_as_float(o1[k]) : 0.f;
              f[e] = x0 + x1;
            }
            *reinterpret_cast<float2*>(dst + 8 * i) = make_float2(f[0], f[1]);
          }
        }
      }
      if (t0 == 0) {
        if (gA < G) {
          p.pm[base + gA] = Mr[0];
          p.pl[base + gA] = Lr[0];
        }
        if (gB < G) {
          p.pm[base + gB] = Mr[1];
          p.pl[base + gB] = Lr[1];
        }
      }
    }
  }
  // (with the in-kernel merge the CTA releases its dependents in fused_merge,
  // once its group's counters are re-armed)
  if (!p.fused) asm volatile("griddepcontrol.launch_dependents;");
  umma::fence_before();
  __syncthreads();
  trace_stamp(4);
  ring_stamp(p, 4);
  if (warp == 1) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, 512);
  }
  if (p.fused) fused_merge(p, sess * nkv + h, j_split, h, G, s_rows);
  ring_stamp(p, 6);
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
int kv_tensor_map(const psk_kv_layout& kv, CUtensorMap* out, int kind) {
  using namespace dattn;
  // small cache keyed by the pool geometry and the box kind
  static CUtensorMap cached[8];
  static psk_kv_layout keys[8] = {};
  static int kinds[8] = {};
  static int next = 0;
  for (int i = 0; i < 8; ++i)
    if (keys[i].base == kv.base && keys[i].n_pages == kv.n_pages && keys[i].page_elems == kv.page_elems &&
        kinds[i] == kind) {
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
  if (kind == KV_BOX2D) {
    cuuint64_t dims[2] = {(cuuint64_t)HD, rows};
    cuuint64_t strides[1] = {(cuuint64_t)HD * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)PT};
    cuuint32_t es[2] = {1, 1};
    r = enc(&cached[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, kv.base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else if (kind == KV_TILE3D) {
    cuuint64_t dims[3] = {64, rows, 2};
    cuuint64_t strides[2] = {(cuuint64_t)HD * 2, 128};
    cuuint32_t box[3] = {64, (cuuint32_t)PT, 2};
    cuuint32_t es[3] = {1, 1, 1};
    r = enc(&cached[i], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, kv.base, dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  } else {
    // (dim, token row, half, K|V): the V tile of a (page, layer, head) sits
    // n_kv_heads tiles after its K tile; KV_PAGE4D_ALL takes all heads' rows
    cuuint64_t dims[4] = {64, rows, 2, 2};
    cuuint64_t strides[3] = {(cuuint64_t)HD * 2, 128, (cuuint64_t)kv.n_kv_heads * PT * HD * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)(kind == KV_PAGE4D_ALL ? PT * kv.n_kv_heads : PT), 2, 2};
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
  kinds[i] = kind;
  *out = cached[i];
  return PSK_OK;
}

}  // namespace psk

using namespace psk::dattn;

extern "C" {

static int sm_count() { return psk::sm_budget(); }

// Launch ring (diagnostics, PSK_TRACE_RING=1): each fan-out launch (captured
// launches included: the slot is fixed at launch / capture time) stamps its
// CTAs' phases into the next of RING_SLOTS slots of RING_CTAS x 8 stamps.
static constexpr int RING_SLOTS = 512, RING_CTAS = 256;
static unsigned long long* g_ring = nullptr;
static int g_ring_n = 0;
static unsigned long long* ring_slot(int ctas) {
  static const bool on = getenv("PSK_TRACE_RING") != nullptr;
  if (!on || ctas > RING_CTAS) return nullptr;
  if (!g_ring) {
    if (cudaMalloc(&g_ring, sizeof(unsigned long long) * RING_SLOTS * RING_CTAS * 8) != cudaSuccess) return nullptr;
    cudaMemset(g_ring, 0, sizeof(unsigned long long) * RING_SLOTS * RING_CTAS * 8);
  }
  return g_ring + (size_t)(g_ring_n++ % RING_SLOTS) * RING_CTAS * 8;
}

int psk_decode_attn_trace_ring(uint64_t* host, int64_t n_u64, int32_t* launches, int32_t* ctas_stride) {
  PSK_CHECK_ARG(launches && ctas_stride, "psk_decode_attn_trace_ring: bad args");
  *launches = g_ring_n;
  *ctas_stride = RING_CTAS;
  if (!g_ring || !host) return PSK_OK;
  const int64_t cap = (int64_t)RING_SLOTS * RING_CTAS * 8;
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  PSK_CUDA_TRY(cudaMemcpy(host, g_ring, sizeof(uint64_t) * (n_u64 < cap ? n_u64 : cap), cudaMemcpyDeviceToHost));
  return PSK_OK;
}

// Partial slots the workspace holds: enough for the caller's fixed splits,
// the stream-K schedule (grid + groups) and the all-heads kernel (one
// wave of (session, split) CTAs: groups x sms / n_sess).
static int64_t ws_slots(const psk_decode_batch* b, int32_t n_kv_heads, int32_t splits) {
  const int64_t groups = (int64_t)b->n_sess * n_kv_heads;
  const int sms = psk::device_sms();  // any budget <= the device count fits
  int64_t slots = (int64_t)sms + groups;
  if (splits > 0 && groups * splits > slots) slots = groups * splits;
  // all-heads kernel: at most 8 waves of CTAs and 4 pages per split (launch)
  const int64_t max_pages = (int64_t)b->max_sess_pages + (int64_t)b->max_rows_per_sess * b->max_row_pages;
  int64_t hsplit = b->n_sess > 0 ? 8 * (int64_t)sms / b->n_sess : 1;
  if (hsplit > max_pages / 4) hsplit = max_pages / 4;
  if (hsplit < 1) hsplit = 1;
  if (groups * hsplit > slots) slots = groups * hsplit;
  return slots;
}

int psk_decode_attn_workspace(const psk_decode_batch* b, int32_t n_kv_heads, int32_t splits,
                              int64_t* bytes) {
  PSK_CHECK_ARG(b && bytes && splits >= 0, "psk_decode_attn_workspace: bad args");
  const int64_t groups = (int64_t)b->n_sess * n_kv_heads;
  // fan-out merge counters at a fixed offset (zero before the first launch;
  // every launch leaves the arrival counts zero, so one workspace serves any
  // batch shape) |
  // partials | CTA directory (+ page total)
  *bytes = CNT_INTS * 4 + ws_slots(b, n_kv_heads, splits) * GMAX * (HD + 2) * 4 + groups * 2 * 4 + 16;
  return PSK_OK;
}

// The all-heads kernel's plan: whether it runs (<= 16 query rows per KV head
// everywhere and at least one (session, head) group per SM), its splits per
// session (one wave of (session, split) CTAs) and whether those CTAs merge
// their session themselves (the wave fits the device: all co-resident).
// Measured at 4k shared tokens x 4 modules (tools/hsplit_ab.py): 32 sessions
// 4 splits 114.5 us vs 5 / 6 / 7 / 8 / 9 splits 142.8 / 124.8 / 118.3 /
// 117.1 / 122.6 us (more than one wave, or more, shorter CTAs that lose to
// their per-CTA prologue); 64 sessions 2 splits 216.9 us, 4 splits 213.1.
// With fewer groups the per-head kernel's finer splits win (8 sessions:
// 42.7 vs 45.8 us; 32 sessions: 152 vs 144 us; 1 session: 12.4 vs 21 us at
// 4k). PSK_ATTN_HSPLIT=n overrides the splits (bounded by the workspace's 8
// waves); PSK_ATTN_MERGE_KERNEL=1 keeps the merge kernel.
static bool heads_plan(const psk_decode_batch* b, int32_t n_q_heads, int32_t n_kv_heads, int32_t splits,
                       int* hsplit, bool* fused) {
  static const bool force_hmma = getenv("PSK_ATTN_HMMA") != nullptr;
  static const bool no_heads = getenv("PSK_ATTN_PER_HEAD") != nullptr;
  static const bool merge_kernel = getenv("PSK_ATTN_MERGE_KERNEL") != nullptr;
  static const int force = getenv("PSK_ATTN_HSPLIT") ? atoi(getenv("PSK_ATTN_HSPLIT")) : 0;
  const int grp = n_q_heads / n_kv_heads;
  const int sms = sm_count();
  const bool use_tc = grp * b->max_rows_per_sess > 32 && !force_hmma;
  if (use_tc || no_heads || splits <= 0 || grp * b->max_rows_per_sess > 16 || n_kv_heads > hk::MAXKV ||
      (int64_t)b->n_sess * n_kv_heads < sms)
    return false;
  const int64_t max_pages = (int64_t)b->max_sess_pages + (int64_t)b->max_rows_per_sess * b->max_row_pages;
  const int64_t hmax = max_pages / 4 > 1 ? max_pages / 4 : 1;
  int h = sms / b->n_sess > 1 ? sms / b->n_sess : 1;
  if (h > hmax) h = (int)hmax;
  if (force > 0 && force <= hmax && b->n_sess * force <= 8 * (int64_t)sms) h = force;
  *hsplit = h;
  *fused = !merge_kernel && (int64_t)b->n_sess * h <= psk::device_sms() &&
           2 * (int64_t)b->n_sess * n_kv_heads <= CNT_INTS;
  return true;
}

// Whether the fan-out (tcgen05) kernel runs and merges its splits itself:
// > 32 query rows per KV head, its (session, head, split) CTAs fit one wave
// (1 CTA per SM, all co-resident for the in-kernel merge).
static bool fanout_fused(const psk_decode_batch* b, int32_t n_q_heads, int32_t n_kv_heads, int32_t splits) {
  static const bool force_hmma = getenv("PSK_ATTN_HMMA") != nullptr;
  static const bool merge_kernel = getenv("PSK_ATTN_MERGE_KERNEL") != nullptr;
  const int grp = n_q_heads / n_kv_heads;
  if (grp * b->max_rows_per_sess <= 32 || force_hmma || merge_kernel) return false;
  const int64_t groups = (int64_t)b->n_sess * n_kv_heads;
  if (splits == 0) splits = (int)(sm_count() / groups) > 1 ? (int)(sm_count() / groups) : 1;
  return groups * splits <= psk::device_sms() && 2 * groups <= CNT_INTS;
}

int psk_decode_attn_kernels(const psk_decode_batch* b, int32_t n_q_heads, int32_t n_kv_heads, int32_t splits,
                            int32_t* n_kernels) {
  PSK_CHECK_ARG(b && n_kernels && n_kv_heads > 0 && n_q_heads % n_kv_heads == 0 && splits >= 0,
                "psk_decode_attn_kernels: bad args");
  int hsplit = 1;
  bool hfused = false;
  const bool heads = heads_plan(b, n_q_heads, n_kv_heads, splits, &hsplit, &hfused);
  *n_kernels = b->n_rows == 0 ? 0 : ((heads ? hfused : fanout_fused(b, n_q_heads, n_kv_heads, splits)) ? 1 : 2);
  return PSK_OK;
}

int psk_decode_attn(const psk_decode_batch* b, const void* q_rot, int32_t n_q_heads, int32_t layer,
                    psk_kv_layout kv, int32_t splits, void* workspace, void* out, void* stream) {
  PSK_CHECK_ARG(b && q_rot && out && workspace && kv.head_dim == HD && kv.page_tokens == PT &&
                    kv.n_pages > 0 && n_q_heads % kv.n_kv_heads == 0 && splits >= 0,
                "psk_decode_attn: bad args");
  const int grp = n_q_heads / kv.n_kv_heads;
  PSK_CHECK_ARG(b->max_rows_per_sess <= MAXR && grp * b->max_rows_per_sess <= GMAX,
                "psk_decode_attn: %d query rows per KV head exceed %d", grp * b->max_rows_per_sess, GMAX);
  if (b->n_rows == 0) return PSK_OK;
  // > 32 query rows per KV head (3-4 m16 tiles): tcgen05 fan-out kernel
  // (32k x 16 modules: 36.7 us vs 48.6 us); up to 32 rows mma.sync is faster
  // (32k x 8: 30.1 vs 32.0 us). PSK_ATTN_HMMA=1 keeps mma.sync everywhere.
  static const bool force_hmma = getenv("PSK_ATTN_HMMA") != nullptr;
  static const bool no_heads = getenv("PSK_ATTN_PER_HEAD") != nullptr;
  const bool use_tc = grp * b->max_rows_per_sess > 32 && !force_hmma;
  const int sms = sm_count();
  const int64_t groups = (int64_t)b->n_sess * kv.n_kv_heads;
  const int64_t slots = ws_slots(b, kv.n_kv_heads, splits);
  int hsplit = 1;
  bool hfused = false;
  const bool use_heads = heads_plan(b, n_q_heads, kv.n_kv_heads, splits, &hsplit, &hfused);
  // stream-K mode (splits == 0) for the mma.sync path when the session
  // tables and one run's page list fit in shared memory; otherwise (and for
  // the tcgen05 path) fixed splits that fit the same workspace
  bool stream_k = false;
  if (splits == 0) {
    const int64_t per_group = (int64_t)b->max_sess_pages + (int64_t)b->max_rows_per_sess * b->max_row_pages;
    const int64_t run_bound = (groups * per_group + sms - 1) / sms + 1;
    stream_k = !use_tc && b->n_sess <= sk::MAXS && run_bound <= sk::MAXP;
    if (!stream_k) splits = (int)(sms / groups) > 1 ? (int)(sms / groups) : 1;  // one wave, fits the slots
  }
  CUtensorMap map;
  const int rc = psk::kv_tensor_map(kv, &map, use_heads ? psk::KV_PAGE4D_ALL : psk::KV_PAGE4D);
  if (rc) return rc;
  Params p;
  p.b = *b;
  p.kv = kv;
  p.q = reinterpret_cast<const __nv_bfloat16*>(q_rot);
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.nq = n_q_heads;
  p.grp = grp;
  p.layer = layer;
  p.ns = stream_k ? 0 : (use_heads ? hsplit : splits);
  // CTAs of the partial kernel
  const int64_t items = stream_k ? sms : (use_heads ? (int64_t)b->n_sess * hsplit : groups * splits);
  p.cnt = reinterpret_cast<unsigned*>(workspace);
  float* ws = reinterpret_cast<float*>(workspace) + CNT_INTS;
  p.pm = ws;
  p.pl = ws + slots * GMAX;
  p.po = ws + 2 * slots * GMAX;
  p.dir = reinterpret_cast<int*>(ws + slots * GMAX * (HD + 2));
  p.sk_grid = sms;
  // fan-out kernel: merge inside the partial kernel when every CTA is
  // co-resident (one CTA per SM); PSK_ATTN_MERGE_KERNEL=1 keeps the kernel
  p.fused = use_tc ? fanout_fused(b, n_q_heads, kv.n_kv_heads, splits) : (use_heads && hfused);

  // The fan-out kernel streams the shared prompt pages before its PDL wait:
  // no kernel of a decode step writes them, and the step's first kernel
  // (embed_rows) waits for all earlier work (prefill, handoff copies) before
  // it lets its dependents launch, so they are complete whenever this kernel
  // runs. 32k x 16 modules 32.9 -> 32.4 us, 8 x 4k x 16 35.3 -> 35.0 us
  // (same box, tools/k6_ab.py). PSK_ATTN_LATE=1 waits first.
  static const bool late = getenv("PSK_ATTN_LATE") != nullptr;
  p.early = !late;
  static const bool stream_only = getenv("PSK_ATTN_STREAM_ONLY") != nullptr;
  p.stream_only = stream_only;
  p.ring = use_tc ? ring_slot((int)items) : nullptr;
  p.scale_log2 = 1.4426950408889634f / sqrtf((float)HD);
  cudaStream_t s = psk::as_stream(stream);
  static bool init = false;
  if (!init) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(decode_attn_partial, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM));
    PSK_CUDA_TRY(cudaFuncSetAttribute(sk::decode_attn_sk, cudaFuncAttributeMaxDynamicSharedMemorySize, sk::SMEM));
    PSK_CUDA_TRY(cudaFuncSetAttribute(hk::decode_attn_heads, cudaFuncAttributeMaxDynamicSharedMemorySize, hk::SMEM));
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
  } else if (stream_k) {
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = sk::SMEM;
    PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, sk::decode_attn_sk, map, p));
  } else if (use_heads) {
    cfg.blockDim = dim3(hk::THREADS);
    cfg.dynamicSmemBytes = hk::SMEM;
    PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, hk::decode_attn_heads, map, p));
  } else {
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = SMEM;
    PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, decode_attn_partial, map, p));
  }
  if (tr) {
    static const char* names_h[] = {"entry", "prologue", "staged", "loop-done", "folded"};  // (stream-K: 0, 1, 3, 4)
    static const char* names_t[] = {"entry", "tmem+bars", "q-staged", "tma-issued", "done"};
    const char* const* names = use_tc ? names_t : names_h;
    psk::trace_report("decode_attn", (int)items, 5, names);
    psk::trace_disarm();
  }
  if (p.fused) return PSK_OK;
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
