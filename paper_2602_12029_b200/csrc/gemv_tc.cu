// K5-TC — grouped decode GEMV on the 5th-gen tensor cores, for 9..64 decode
// rows per module (the co-batched fan-out regime: many sessions x modules).
//
// Same contract as psk_gemv (gemv.cu): for each module i and each of its rows
// r, y[r, n] = sum_k x[r, k] * W_i[n, k], fused epilogues. At <= 8 rows per
// module the mma.sync kernel streams weights at the HBM roofline; above that
// its register-resident x fragments and cross-warp reductions make it
// compute/L2-bound (16 rows: ~1.2x, 32 rows: ~2.7x the weight-stream time).
// Here the skinny GEMM D[128 weight rows, M rows] = W_blk . X^T runs as
// tcgen05.mma M=128, N=MN (16/32/64), K=16 with the accumulator in TMEM: no
// cross-warp reduction, x is staged once per k-chunk by TMA, and the kernel
// is a pure TMA weight stream again.
//
// Persistent, one CTA per SM, 6 warps:
//   warp 0   TMA producer: per 64-column k-chunk one 128x64 weight box
//            (16 KiB, SW128) per 128-row block + one MNx64 x box; 2-4
//            chunks per ring stage behind one mbarrier (216 KiB ring); the
//            weight boxes of the first ring fill are issued before the PDL
//            wait (weights never depend on the previous kernel)
//   warp 1   MMA issuer (one lane): 4 x tcgen05.mma per chunk into one of two
//            TMEM accumulators (double-buffered across segments)
//   warps 2-5  epilogue: tcgen05.ld 32x32b (thread = weight row, one column
//            per activation row), fused store / residual add / SiLU*mul /
//            the decode QKV epilogue (RoPE on q and k, q_rot out, k and v
//            appended to each row's private KV page: a 128-row unit is one
//            head, the rotate-half partner dims swap through shared memory)
// Work unit = (module, 128-row weight block) x K; the CTAs split the
// (unit, 64-column chunk) space stream-K style (below).
//
// Replaces the per-module dense projections of the reference decode forward
// (frontend/src/model.ts:298-306 q/k/v, :318 o-proj, :322-323 MLP, :334
// logits), for all decode modules of a step in one launch.
#include "common.cuh"
#include "tma.cuh"
#include "umma.cuh"

namespace psk {
namespace gemv_tc {

constexpr int BN = 128;             // weight rows per unit (UMMA M)
constexpr int BK = 64;              // columns per k-chunk (one 128 B swizzle atom)
constexpr int A_BYTES = BN * BK * 2;  // 16 KiB
constexpr int THREADS = 192;
constexpr int MAXMOD = 16;
constexpr int RING_BYTES = 216 * 1024;
// k-chunks per ring stage: the producer issues CH weight boxes back to back
// per mbarrier (tools/bw_probe.cu: 128x64 SW128 boxes stream at 6.35 TB/s
// one per stage, 6.97-7.0 TB/s three or four per stage)
// UW = 128-row weight blocks per work unit. UW = 2 (N % 256 == 0): one x box
// per k-chunk serves two M=128 MMAs into two TMEM accumulators, halving the
// x traffic and putting 192 KiB of weights in flight in two stages.
template <int MN, int UW>
struct Cfg {
  static constexpr int CH = UW == 2 ? (MN <= 32 ? 3 : 2) : (MN <= 16 ? 4 : (MN <= 32 ? 3 : 2));
  static constexpr int B_BYTES = MN * BK * 2;
  static constexpr int STAGE = CH * (UW * A_BYTES + B_BYTES);  // [CH x UW weight boxes][CH x boxes]
  static constexpr int STAGES = RING_BYTES / STAGE;
  static constexpr int SMEM = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int TMEM_COLS = 2 * UW * MN < 32 ? 32 : 2 * UW * MN;
  static_assert(STAGE % 1024 == 0, "SW128 tiles need 1 KiB alignment");
};

struct Maps {
  CUtensorMap w[MAXMOD];  // per-module weight [N][K], box {64, 128}
  CUtensorMap x;          // activations [n_rows][K], box {64, MN}
};

// EPI_QKV_ROPE (psk_gemv_tc_qkv_rope): the decode step's QKV projection with
// RoPE + KV append fused (replaces psk_gemv_tc(STORE_F32) + psk_rope_append).
// EPI_RESID_NORM (psk_gemv_tc_resid_norm): residual add + the next RMSNorm
// (replaces psk_gemv_tc(RESID_ADD) + psk_rmsnorm_rows); one CTA per whole
// unit, the module's units meet at a grid barrier to sum their rows' squares.
constexpr int EPI_QKV_ROPE = 16;
constexpr int EPI_RESID_NORM = 17;
constexpr int NORM_MAXNB = 64;  // 128-row units per module (N <= 8192)
struct RopeArgs {
  psk_decode_batch b;
  psk_kv_layout kv;
  const float* rope;       // [max_pos][64][2] (cos, sin)
  __nv_bfloat16* q_rot;    // [n_rows][nq][128]
  int nq, layer;
  // EPI_RESID_NORM
  const __nv_bfloat16* const* gamma;  // per module of the batch
  __nv_bfloat16* xn;                  // [n_rows][N] bf16(h * rsqrt(mean(h^2) + eps) * gamma)
  float eps;
  float* ssq;                         // [MAXMOD][64 rows][NORM_MAXNB] per-unit partial sums of squares
  unsigned* cnt;                      // [MAXMOD][2] arrived / departed (zero between launches)
  unsigned long long* ring;           // diagnostics (PSK_TRACE_RING=1): this launch's [CTA][8] stamps
  int ring_n;                         //   and its N (which projection)
};

// Launch-ring stamp (%globaltimer) of phase k by the calling thread
__device__ __forceinline__ void gring(const RopeArgs& ra, int k) {
  if (ra.ring != nullptr) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    ra.ring[(size_t)blockIdx.x * 8 + k] = v;
  }
}

__device__ __forceinline__ void tmem_ld32_cols(uint32_t taddr, float* v) {
  uint32_t r[32];
  umma::ld32_async(taddr, r);
  umma::wait_ld();
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld16_cols(uint32_t taddr, float* v) { umma::ld16(taddr, v); }

// Stream-K work split: the (unit, k-chunk) space is cut into gridDim.x equal
// runs of chunks, so every CTA streams the same number of weight bytes
// whatever the unit count (o/down: 128 units, qkv: 192, gate/up: 896 on 148
// SMs). A run is a sequence of segments, one per unit it touches. The segment
// holding a unit's chunk 0 is the unit's owner (it is the run's LAST segment
// when the unit continues into the next runs); a segment without chunk 0 is
// a contributor and is always the run's FIRST segment, so each CTA has at
// most one contributor segment (one fp32 partial slot [MN][128] + a flag).
// Contributors publish early (start of their run); the owner reaches the
// unit at the end of its run, sums its accumulator and the partials of the
// following CTAs in a fixed order (bit-reproducible), then runs the fused
// epilogue. Waits only point to higher CTAs, whose first segments never
// wait, and all CTAs are co-resident (grid <= SMs): no deadlock.
struct Seg {
  int unit, k0, k1;  // chunks [k0, k1) of `unit`
};

__device__ __forceinline__ int run_begin(int cta, int64_t total, int grid) {
  return (int)((int64_t)cta * total / grid);
}

template <int MN, int EPI, int UW>
__global__ void __launch_bounds__(THREADS, 1)
    gemv_tc_kernel(const __grid_constant__ Maps maps, const int32_t* __restrict__ mrs, int n_mod, int N, int K,
                   void* __restrict__ out, float* __restrict__ part, int* __restrict__ flags,
                   const __grid_constant__ RopeArgs ra) {
  using C = Cfg<MN, UW>;
  static_assert((EPI != EPI_QKV_ROPE && EPI != EPI_RESID_NORM) || UW == 1, "one 128-row block per unit");
  constexpr int UB = UW * BN;  // weight rows per unit
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  // EPI_QKV_ROPE: [MN][128] fp32 exchange tile + per-row (pos, page, token)
  // (+ at MN = 32 the rows' RoPE (cos, sin) [MN][64], staged under the MMAs)
  constexpr bool CS_SMEM = EPI == EPI_QKV_ROPE && MN == 32;
  float* xch = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE + 256);
  int* meta = reinterpret_cast<int*>(xch + MN * BN);
  float2* cs_s = reinterpret_cast<float2*>(meta + 4 * MN);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nb = N / UB;
  const int kcn = (K + BK - 1) / BK;
  const int64_t total = (int64_t)n_mod * nb * kcn;
  const int cta = blockIdx.x, grid = gridDim.x;
  const int c0 = run_begin(cta, total, grid), c1 = run_begin(cta + 1, total, grid);
  // segment iterator over [c0, c1)
  auto seg_at = [&](int c) -> Seg {
    const int unit = c / kcn;
    const int k0 = c % kcn;
    const int k1 = min(kcn, k0 + (c1 - c));
    return Seg{unit, k0, k1};
  };
  auto live = [&](int unit) -> bool {
    const int mod = unit / nb;
    return mrs[mod + 1] > mrs[mod];
  };

  if (threadIdx.x == 0) {
    gring(ra, 0);
    for (int s = 0; s < C::STAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      tma::mbar_init(&tfull[s], 1);
      tma::mbar_init(&tempty[s], 128);
    }
    tma::fence_mbar_init();
  }
  if (warp == 1) umma::tmem_alloc(tmem_slot, C::TMEM_COLS);
  umma::fence_before();
  __syncthreads();
  umma::fence_after();
  pdl_trigger();  // the next kernel may start streaming its weights as our CTAs drain
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) gring(ra, 1);

  if (warp == 0) {
    // warp-converged (all lanes, warp-uniform operands, one elected lane
    // issues): from if (lane == 0) every TMA / MMA became an R2UR waterfall loop
    {
      if (lane == 0) {
        for (int m = 0; m < n_mod && m < MAXMOD; ++m) tma::prefetch_map(&maps.w[m]);
        tma::prefetch_map(&maps.x);
      }
      __syncwarp();
      // x rows come from the previous kernel: the first ring fill issues the
      // weight boxes at once and the x boxes after the PDL wait
      int pend_k[C::STAGES], pend_n[C::STAGES], pend_row[C::STAGES];
      int npend = 0;
      bool waited = false;
      int j = 0;  // stage counter
      auto load_x = [&](int s, int k0c, int n, int row) {
        for (int b = 0; b < n; ++b)
          tma::load_2d_e(&maps.x, &full[s], smem + s * C::STAGE + C::CH * UW * A_BYTES + b * C::B_BYTES,
                       (k0c + b) * BK, row);
      };
      for (int c = c0; c < c1;) {
        const Seg sg = seg_at(c);
        c += sg.k1 - sg.k0;
        if (!live(sg.unit)) continue;  // module without rows this step
        const int mod = sg.unit / nb, blk = sg.unit % nb;
        const int xb = mrs[mod];
        for (int kc = sg.k0; kc < sg.k1; kc += C::CH, ++j) {
          const int n = min(C::CH, sg.k1 - kc);
          const int s = j % C::STAGES;
          if (!waited && j == C::STAGES) {
            pdl_wait();
            if (lane == 0) gring(ra, 3);
            for (int i = 0; i < npend; ++i) load_x(i, pend_k[i], pend_n[i], pend_row[i]);
            waited = true;
          }
          tma::mbar_wait(&empty[s], ((j / C::STAGES) & 1) ^ 1);
          tma::mbar_expect_tx_e(&full[s], n * (UW * A_BYTES + C::B_BYTES));
          unsigned char* st = smem + s * C::STAGE;
          for (int b = 0; b < n; ++b)
            for (int u = 0; u < UW; ++u)
              tma::load_2d_e(&maps.w[mod], &full[s], st + (b * UW + u) * A_BYTES, (kc + b) * BK, blk * UB + u * BN);
          if (j == 0 && lane == 0) gring(ra, 2);
          if (waited) {
            load_x(s, kc, n, xb);
          } else {
            pend_k[npend] = kc;
            pend_n[npend] = n;
            pend_row[npend] = xb;
            ++npend;
          }
        }
      }
      if (!waited) {
        pdl_wait();
        if (lane == 0) gring(ra, 3);
        for (int i = 0; i < npend; ++i) load_x(i, pend_k[i], pend_n[i], pend_row[i]);
      }
      if (lane == 0) gring(ra, 4);
    }
  } else if (warp == 1) {
    {
      constexpr uint32_t idesc = umma::idesc_bf16(BN, MN, false);
      int j = 0, it = 0;
      for (int c = c0; c < c1;) {
        const Seg sg = seg_at(c);
        c += sg.k1 - sg.k0;
        if (!live(sg.unit)) continue;
        const int acc = it & 1;
        tma::mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        umma::fence_after();
        const uint32_t tacc = tmem + acc * UW * MN;
        for (int kc = sg.k0; kc < sg.k1; kc += C::CH, ++j) {
          const int n = min(C::CH, sg.k1 - kc);
          const int s = j % C::STAGES;
          tma::mbar_wait(&full[s], (j / C::STAGES) & 1);
          umma::fence_after();
          const uint32_t a = tma::sa(smem + s * C::STAGE);
          for (int b = 0; b < n; ++b) {
            const uint64_t db = umma::desc_k_sw128(a + C::CH * UW * A_BYTES + b * C::B_BYTES);
#pragma unroll
            for (int u = 0; u < UW; ++u) {
              const uint64_t da = umma::desc_k_sw128(a + (b * UW + u) * A_BYTES);
#pragma unroll
              for (int k = 0; k < BK / 16; ++k)
                umma::mma_e(tacc + u * MN, da + 2 * k, db + 2 * k, idesc, (kc + b != sg.k0 || k != 0) ? 1u : 0u);
            }
          }
          umma::commit_e(&empty[s]);
        }
        umma::commit_e(&tfull[acc]);
        ++it;
      }
      if (lane == 0) gring(ra, 5);
    }
  } else {
    // epilogue: warp w reads TMEM lane quarter w % 4 = weight rows 32q..32q+31
    const int q = warp & 3;
    const int r = q * 32 + lane;  // weight row within the unit
    pdl_wait();                   // out (residual stream) is written by earlier kernels
    int it = 0;
    for (int c = c0; c < c1;) {
      const Seg sg = seg_at(c);
      c += sg.k1 - sg.k0;
      if (!live(sg.unit)) continue;
      const int mod = sg.unit / nb, blk = sg.unit % nb;
      const int xb = mrs[mod], M = mrs[mod + 1] - xb;
      const bool owner = sg.k0 == 0;
      const int acc = it & 1;
      bool waited_tfull = false;
      if (EPI == EPI_QKV_ROPE && owner) {
        // the previous unit's readers of xch / meta are done; stage this
        // unit's row positions and append slots (sess_len + priv_len, page)
        named_barrier_sync(3, 128);
        const int t = threadIdx.x - 64;
        if (t < M) {
          const int row = xb + t, idx = ra.b.priv_len[row];
          meta[3 * t] = ra.b.sess_len[ra.b.row_sess[row]] + idx;
          meta[3 * t + 1] = ra.b.row_pages[(int64_t)row * ra.b.max_row_pages + idx / 16];
          meta[3 * t + 2] = idx % 16;
        }
        if (CS_SMEM && blk < ra.nq + ra.kv.n_kv_heads) {  // q / k head: stage its rows' (cos, sin)
          named_barrier_sync(3, 128);
          const float2* rope2 = reinterpret_cast<const float2*>(ra.rope);
          for (int e = t; e < M * 64; e += 128) cs_s[e] = __ldg(rope2 + (int64_t)meta[3 * (e >> 6)] * 64 + (e & 63));
        }
      }
#pragma unroll 1
      for (int u = 0; u < UW; ++u) {
      const int n = blk * UB + u * BN + r;
      float v[MN];
      // residual prefetch: its latency overlaps this segment's MMAs
      if ((EPI == PSK_EPI_RESID_ADD || EPI == EPI_RESID_NORM) && owner) {
#pragma unroll
        for (int m = 0; m < MN; ++m)
          v[m] = m < M ? reinterpret_cast<const float*>(out)[(int64_t)(xb + m) * N + n] : 0.f;
      } else {
#pragma unroll
        for (int m = 0; m < MN; ++m) v[m] = 0.f;
      }
      if (!waited_tfull) {
        tma::mbar_wait(&tfull[acc], (it >> 1) & 1);
        umma::fence_after();
        waited_tfull = true;
      }
      {
        const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + acc * UW * MN + u * MN;
        float a[MN];
        if (MN == 16) {
          umma::ld16(tacc, a);
        } else {
#pragma unroll
          for (int cc = 0; cc < MN / 32; ++cc) {
            uint32_t t[32];
            umma::ld32_async(tacc + cc * 32, t);
            umma::wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) a[cc * 32 + i] = __uint_as_float(t[i]);
          }
        }
        if (u == UW - 1) {
          umma::fence_before();
          tma::mbar_arrive(&tempty[acc]);  // the MMA of segment it+2 may overwrite it
        }
        if (!owner) {
          // contributor (this run's first segment): publish the fp32 partial
          float* slot = part + ((int64_t)cta * UW + u) * MN * BN;
#pragma unroll
          for (int m = 0; m < MN; ++m) slot[m * BN + r] = a[m];
          if (u == UW - 1) {
            __threadfence();
            named_barrier_sync(2, 128);
            if (threadIdx.x == 64)
              asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(flags + cta), "r"(1) : "memory");
          }
          continue;
        }
        // owner: own accumulator + partials of the following runs, fixed order
        const int64_t unit_end = (int64_t)(sg.unit + 1) * kcn;
        if (sg.k1 < kcn) {
          for (int j2 = cta + 1; j2 < grid && run_begin(j2, total, grid) < unit_end; ++j2) {
            if (u == 0) {
              if (threadIdx.x == 64) {
                int f = 0;
                do {
                  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(f) : "l"(flags + j2) : "memory");
                } while (f == 0);
                flags[j2] = 0;  // consumed: ready for the next launch
              }
              named_barrier_sync(2, 128);
            }
            const float* slot = part + ((int64_t)j2 * UW + u) * MN * BN;
#pragma unroll
            for (int m = 0; m < MN; ++m) a[m] += __ldcg(slot + m * BN + r);
          }
        }
#pragma unroll
        for (int m = 0; m < MN; ++m) v[m] += a[m];
      }
      if (EPI == EPI_QKV_ROPE) {
        const int nkv = ra.kv.n_kv_heads, hd = blk;  // unit = head: q heads, then k, then v
        if (hd < ra.nq + nkv) {
#pragma unroll
          for (int m = 0; m < MN; ++m) xch[m * BN + r] = v[m];
        }
        named_barrier_sync(3, 128);  // xch and meta visible
        const int i = r & 63;
        const bool vhead = hd >= ra.nq + nkv;
        const float2* rope2 = reinterpret_cast<const float2*>(ra.rope);
        // 8 rows at a time: their (cos, sin) loads are all in flight before
        // the first store (stores to q_rot / the pages may alias the table
        // for the compiler, so interleaving would serialise the loads)
#pragma unroll
        for (int m0 = 0; m0 < MN; m0 += 8) {
          if (m0 >= M) break;
          float2 cs[8];
#pragma unroll
          for (int j = 0; j < 8; ++j)
            cs[j] = (vhead || m0 + j >= M) ? make_float2(0.f, 0.f)
                    : CS_SMEM             ? cs_s[(m0 + j) * 64 + i]
                                          : __ldg(rope2 + (int64_t)meta[3 * (m0 + j)] * 64 + i);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int m = m0 + j;
            if (m >= M) break;
            const int page = meta[3 * m + 1], tok = meta[3 * m + 2];
            if (vhead) {
              kv_row(ra.kv, page, ra.layer, 1, hd - ra.nq - nkv, tok)[r] = f2bf(v[m]);
              continue;
            }
            const float o = xch[m * BN + (r ^ 64)];
            float y1, y2;
            if (r < 64)
              rope_pair(v[m], o, cs[j].x, cs[j].y, y1, y2);
            else
              rope_pair(o, v[m], cs[j].x, cs[j].y, y1, y2);
            const __nv_bfloat16 y = f2bf(r < 64 ? y1 : y2);
            if (hd < ra.nq)
              ra.q_rot[((int64_t)(xb + m) * ra.nq + hd) * BN + r] = y;
            else
              kv_row(ra.kv, page, ra.layer, 0, hd - ra.nq, tok)[r] = y;
          }
        }
      } else if (EPI == PSK_EPI_SILU_MUL) {
        // rows interleaved [gate 8 | up 8]: the up row of gate row n is n + 8,
        // held by lane + 8 of this warp
        const bool gate = (r & 15) < 8;
        const int o = (blk * UB + u * BN + (r & ~15)) / 2 + (r & 7);
#pragma unroll
        for (int m = 0; m < MN; ++m) {
          const float up = __shfl_down_sync(0xffffffffu, v[m], 8);
          if (gate && m < M) {
            const float g = v[m];
            reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)(xb + m) * (N / 2) + o] =
                f2bf(g / (1.f + __expf(-g)) * up);
          }
        }
      } else {
#pragma unroll
        for (int m = 0; m < MN; ++m) {
          if (m >= M) break;
          const int64_t o = (int64_t)(xb + m) * N + n;
          if (EPI == PSK_EPI_STORE_BF16) reinterpret_cast<__nv_bfloat16*>(out)[o] = f2bf(v[m]);
          if (EPI == PSK_EPI_STORE_F32 || EPI == PSK_EPI_RESID_ADD || EPI == EPI_RESID_NORM)
            reinterpret_cast<float*>(out)[o] = v[m];
        }
        if (EPI == EPI_RESID_NORM) {
          // this unit's 128 features of each row: sum of squares -> ssq; then,
          // once every unit of the module has published (grid barrier: all
          // CTAs co-resident, one per unit), each row's rstd from the nb
          // partials in a fixed order and the normalised features -> xn
          float* red = xch;  // [4 lane quarters][MN]
#pragma unroll
          for (int m = 0; m < MN; ++m) {
            float sq = m < M ? v[m] * v[m] : 0.f;
            sq = warp_sum(sq);
            if (lane == 0) red[q * MN + m] = sq;
          }
          named_barrier_sync(3, 128);
          const int t = threadIdx.x - 64;
          float* part = ra.ssq + (int64_t)mod * 64 * NORM_MAXNB;
          if (t < M) part[t * NORM_MAXNB + blk] = (red[t] + red[MN + t]) + (red[2 * MN + t] + red[3 * MN + t]);
          named_barrier_sync(3, 128);
          unsigned* cnt = ra.cnt + 2 * mod;
          if (threadIdx.x == 64) {
            __threadfence();
            atomicAdd(cnt, 1u);
            unsigned arrived;
            do {
              asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(arrived) : "l"(cnt) : "memory");
            } while (arrived < (unsigned)nb);
            __threadfence();
          }
          named_barrier_sync(3, 128);
          if (t < M) {
            float tot = 0.f;
            for (int b = 0; b < nb; ++b) tot += __ldcg(part + t * NORM_MAXNB + b);
            red[t] = rsqrtf(tot / (float)N + ra.eps);
          }
          named_barrier_sync(3, 128);
          const float gm = bf2f(ra.gamma[mod][n]);
#pragma unroll
          for (int m = 0; m < MN; ++m) {
            if (m >= M) break;
            ra.xn[(int64_t)(xb + m) * N + n] = f2bf(v[m] * red[m] * gm);
          }
          named_barrier_sync(3, 128);  // red reads done before a next unit (none: one unit per CTA)
          if (threadIdx.x == 64 && atomicAdd(cnt + 1, 1u) == (unsigned)nb - 1) {  // every unit has left the wait
            cnt[0] = 0;
            cnt[1] = 0;
          }
        }
      }
      }  // u
      ++it;
    }
    if (threadIdx.x == 64) gring(ra, 6);
  }
  umma::fence_before();
  __syncthreads();
  if (warp == 1) {
    umma::fence_after();
    umma::tmem_dealloc(tmem, C::TMEM_COLS);
  }
  if (threadIdx.x == 0) gring(ra, 7);
}

// ------------------------------------------------------------ host side --

static int sm_count();
static unsigned long long* ring_slot(int N, int grid);

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult qr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) == cudaSuccess &&
        qr == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// bf16 [rows][cols] row-major, [box_rows x 64] SW128 boxes
static int make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int box_rows,
                    CUtensorMapL2promotion promo) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PSK_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, promo,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("psk_gemv_tc: cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PSK_ECUDA;
  }
  return PSK_OK;
}

static int sm_count() { return psk::sm_budget(); }

// Launch ring (diagnostics, PSK_TRACE_RING=1): every launch (captured ones
// included: the slot is fixed at launch / capture time) stamps its CTAs'
// phases into the next of RING_SLOTS slots of RING_CTAS x 8 stamps; the
// slot's N and grid are kept on the host.
static constexpr int RING_SLOTS = 1024, RING_CTAS = 160;
static unsigned long long* g_ring = nullptr;
static int g_ring_n = 0;
static int g_ring_meta[RING_SLOTS][2];
static unsigned long long* ring_slot(int N, int grid) {
  static const bool on = getenv("PSK_TRACE_RING") != nullptr;
  if (!on || grid > RING_CTAS) return nullptr;
  if (!g_ring) {
    if (cudaMalloc(&g_ring, sizeof(unsigned long long) * RING_SLOTS * RING_CTAS * 8) != cudaSuccess) return nullptr;
    cudaMemset(g_ring, 0, sizeof(unsigned long long) * RING_SLOTS * RING_CTAS * 8);
  }
  const int slot = g_ring_n++ % RING_SLOTS;
  g_ring_meta[slot][0] = N;
  g_ring_meta[slot][1] = grid;
  return g_ring + (size_t)slot * RING_CTAS * 8;
}

constexpr int FLAG_BYTES = 4096;  // one int per CTA (<= 1024 SMs)

template <int MN, int EPI, int UW>
static int launch_uw(const void* x, int n_rows, int K, const void* const* W_host, const int32_t* mrs, int n_mod,
                  int N, void* out, void* ws, cudaStream_t s, const RopeArgs& ra = RopeArgs{}) {
  Maps maps;
  for (int m = 0; m < n_mod; ++m) {
    int rc = make_map(&maps.w[m], W_host[m], N, K, BN, CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
    if (rc) return rc;
  }
  int rc = make_map(&maps.x, x, n_rows, K, MN, CU_TENSOR_MAP_L2_PROMOTION_L2_128B);
  if (rc) return rc;
  auto k = gemv_tc_kernel<MN, EPI, UW>;
  // + the QKV epilogue's exchange tile and row table
  constexpr int smem_bytes = Cfg<MN, UW>::SMEM + (EPI == EPI_QKV_ROPE ? MN * BN * 4 + MN * 4 * 4 : 0) +
                             (EPI == EPI_QKV_ROPE && MN == 32 ? MN * 64 * 8 : 0) +
                             (EPI == EPI_RESID_NORM ? 4 * MN * 4 : 0);
  static_assert(smem_bytes <= 232448, "shared memory");
  static bool attr = false;
  if (!attr) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes));
    attr = true;
  }
  const int sms = sm_count();
  const int64_t units = (int64_t)n_mod * (N / (UW * BN));
  const int64_t chunks = units * ((K + BK - 1) / BK);
  int grid = chunks < sms ? (int)chunks : sms;
  // <= one unit per SM: one CTA per whole unit, no stream-K split and no
  // partial reduction (o-proj at 32 rows/module 26.6 -> 24.8 us, down 76.0 ->
  // 73.2 us); above that the stream-K split balances the SMs (qkv's 192
  // units as 96 CTAs x 2 measured 35.0 -> 37.8 us). PSK_GEMV_GRID=0: always
  // stream-K.
  static const bool whole_units = !(getenv("PSK_GEMV_GRID") && getenv("PSK_GEMV_GRID")[0] == '0');
  if (whole_units && units <= sms) grid = (int)units;
  int* flags = reinterpret_cast<int*>(ws);
  float* part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + FLAG_BYTES);
  RopeArgs rr = ra;
  rr.ring = ring_slot(N, grid);
  rr.ring_n = N;
  PSK_CUDA_TRY(psk::launch_pdl(k, dim3(grid), dim3(THREADS), (size_t)smem_bytes, s, maps, mrs, n_mod, N, K,
                               out, part, flags, rr));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

template <int MN, int EPI>
static int launch(const void* x, int n_rows, int K, const void* const* W_host, const int32_t* mrs, int n_mod,
                  int N, void* out, void* ws, cudaStream_t s) {
  // two 128-row blocks per unit only pay at <= 16 rows per module on the large
  // projections (gate/up 145.6 -> 142.8 us, LM head 642 -> 610 us); at 32 and
  // 64 rows, and for the 4096/6144-row projections, the coarser units lose
  // (gate/up at 32 rows: 146.1 -> 151.6 us)
  if (MN == 16 && N % (2 * BN) == 0 && N >= 16384)
    return launch_uw<MN, EPI, 2>(x, n_rows, K, W_host, mrs, n_mod, N, out, ws, s);
  return launch_uw<MN, EPI, 1>(x, n_rows, K, W_host, mrs, n_mod, N, out, ws, s);
}

template <int MN>
static int dispatch(int epi, const void* x, int n_rows, int K, const void* const* W, const int32_t* mrs,
                    int n_mod, int N, void* out, void* ws, cudaStream_t s) {
  switch (epi) {
    case PSK_EPI_STORE_BF16: return launch<MN, PSK_EPI_STORE_BF16>(x, n_rows, K, W, mrs, n_mod, N, out, ws, s);
    case PSK_EPI_STORE_F32: return launch<MN, PSK_EPI_STORE_F32>(x, n_rows, K, W, mrs, n_mod, N, out, ws, s);
    case PSK_EPI_RESID_ADD: return launch<MN, PSK_EPI_RESID_ADD>(x, n_rows, K, W, mrs, n_mod, N, out, ws, s);
    case PSK_EPI_SILU_MUL: return launch<MN, PSK_EPI_SILU_MUL>(x, n_rows, K, W, mrs, n_mod, N, out, ws, s);
  }
  set_error("psk_gemv_tc: unknown epilogue %d", epi);
  return PSK_EINVAL;
}

}  // namespace gemv_tc
}  // namespace psk

static int64_t part_bytes() { return (int64_t)psk::device_sms() * 2 * 64 * psk::gemv_tc::BN * 4; }  // UW <= 2 x MN <= 64

extern "C" int psk_gemv_tc_trace_ring(uint64_t* host, int64_t n_u64, int32_t* meta, int32_t* launches,
                                      int32_t* ctas_stride) {
  using namespace psk::gemv_tc;
  PSK_CHECK_ARG(launches && ctas_stride, "psk_gemv_tc_trace_ring: bad args");
  *launches = g_ring_n;
  *ctas_stride = RING_CTAS;
  if (!g_ring || !host) return PSK_OK;
  const int64_t cap = (int64_t)RING_SLOTS * RING_CTAS * 8;
  PSK_CUDA_TRY(cudaDeviceSynchronize());
  PSK_CUDA_TRY(cudaMemcpy(host, g_ring, sizeof(uint64_t) * (n_u64 < cap ? n_u64 : cap), cudaMemcpyDeviceToHost));
  if (meta)
    for (int i = 0; i < RING_SLOTS; ++i) {
      meta[2 * i] = g_ring_meta[i][0];
      meta[2 * i + 1] = g_ring_meta[i][1];
    }
  return PSK_OK;
}

extern "C" int psk_gemv_tc_workspace(int64_t* bytes) {
  PSK_CHECK_ARG(bytes != nullptr, "psk_gemv_tc_workspace: null out");
  using namespace psk::gemv_tc;
  // flags | stream-K partials | RMSNorm-epilogue counters + partial sums of squares
  *bytes = FLAG_BYTES + part_bytes() + 256 + (int64_t)MAXMOD * 64 * NORM_MAXNB * 4;
  return PSK_OK;
}

extern "C" int psk_gemv_tc_resid_norm(const void* x, int32_t n_rows, int32_t K, const void* const* W_host,
                                      const int32_t* mod_row_start, int32_t n_mod, int32_t max_rows_per_mod,
                                      int32_t N, float* h, const void* const* gamma, const int32_t* row_mod,
                                      float eps, void* xn, void* workspace, void* stream) {
  using namespace psk::gemv_tc;
  PSK_CHECK_ARG(x && W_host && mod_row_start && h && gamma && xn && workspace && n_rows >= 0 && K > 0 &&
                    K % 64 == 0 && n_mod > 0 && n_mod <= MAXMOD && N > 0 && N % BN == 0,
                "psk_gemv_tc_resid_norm: bad args");
  if (n_rows == 0) return PSK_OK;
  const int maxm = max_rows_per_mod > 0 ? max_rows_per_mod : n_rows;
  cudaStream_t s = psk::as_stream(stream);
  static const bool whole_units = !(getenv("PSK_GEMV_GRID") && getenv("PSK_GEMV_GRID")[0] == '0');
  const bool fused = whole_units && (int64_t)n_mod * (N / BN) <= sm_count() && N / BN <= NORM_MAXNB && maxm <= 64;
  if (!fused) {  // the stream-K split (or > 64 rows): residual GEMV, then the norm kernel
    const int rc = psk_gemv_tc(x, n_rows, K, W_host, mod_row_start, n_mod, max_rows_per_mod, N, PSK_EPI_RESID_ADD,
                               h, workspace, stream);
    return rc ? rc : psk_rmsnorm_rows(h, n_rows, N, gamma, row_mod, eps, xn, stream);
  }
  RopeArgs ra{};
  ra.gamma = reinterpret_cast<const __nv_bfloat16* const*>(gamma);
  ra.xn = reinterpret_cast<__nv_bfloat16*>(xn);
  ra.eps = eps;
  char* w = reinterpret_cast<char*>(workspace) + FLAG_BYTES + part_bytes();
  ra.cnt = reinterpret_cast<unsigned*>(w);
  ra.ssq = reinterpret_cast<float*>(w + 256);
  if (maxm <= 16) return launch_uw<16, EPI_RESID_NORM, 1>(x, n_rows, K, W_host, mod_row_start, n_mod, N, h, workspace, s, ra);
  if (maxm <= 32) return launch_uw<32, EPI_RESID_NORM, 1>(x, n_rows, K, W_host, mod_row_start, n_mod, N, h, workspace, s, ra);
  return launch_uw<64, EPI_RESID_NORM, 1>(x, n_rows, K, W_host, mod_row_start, n_mod, N, h, workspace, s, ra);
}

extern "C" int psk_gemv_tc_qkv_rope(const void* x, int32_t K, const void* const* W_host, const psk_decode_batch* b,
                                    int32_t max_rows_per_mod, int32_t n_q_heads, const float* rope, int32_t layer,
                                    psk_kv_layout kv, void* q_rot, void* workspace, void* stream) {
  using namespace psk::gemv_tc;
  PSK_CHECK_ARG(x && W_host && b && rope && q_rot && workspace && K > 0 && K % 64 == 0 && b->n_mod > 0 &&
                    b->n_mod <= MAXMOD && kv.head_dim == BN && kv.page_tokens == 16 && n_q_heads > 0,
                "psk_gemv_tc_qkv_rope: bad args (K %% 64 == 0, 1..%d modules, head_dim 128, 16-token pages)",
                MAXMOD);
  if (b->n_rows == 0) return PSK_OK;
  const int maxm = max_rows_per_mod > 0 ? max_rows_per_mod : b->n_rows;
  const int N = (n_q_heads + 2 * kv.n_kv_heads) * BN;
  RopeArgs ra;
  ra.b = *b;
  ra.kv = kv;
  ra.rope = rope;
  ra.q_rot = reinterpret_cast<__nv_bfloat16*>(q_rot);
  ra.nq = n_q_heads;
  ra.layer = layer;
  cudaStream_t s = psk::as_stream(stream);
  const int32_t* mrs = b->mod_row_start;
  if (maxm <= 16)
    return launch_uw<16, EPI_QKV_ROPE, 1>(x, b->n_rows, K, W_host, mrs, b->n_mod, N, q_rot, workspace, s, ra);
  if (maxm <= 32)
    return launch_uw<32, EPI_QKV_ROPE, 1>(x, b->n_rows, K, W_host, mrs, b->n_mod, N, q_rot, workspace, s, ra);
  if (maxm <= 64)
    return launch_uw<64, EPI_QKV_ROPE, 1>(x, b->n_rows, K, W_host, mrs, b->n_mod, N, q_rot, workspace, s, ra);
  psk::set_error("psk_gemv_tc_qkv_rope: more than 64 rows per module (%d)", maxm);
  return PSK_EINVAL;
}

extern "C" int psk_gemv_tc(const void* x, int32_t n_rows, int32_t K, const void* const* W_host,
                           const int32_t* mod_row_start, int32_t n_mod, int32_t max_rows_per_mod, int32_t N,
                           int32_t epilogue, void* out, void* workspace, void* stream) {
  using namespace psk::gemv_tc;
  PSK_CHECK_ARG(x && W_host && mod_row_start && out && workspace && n_rows >= 0 && K > 0 && K % 64 == 0 &&
                    n_mod > 0 && n_mod <= MAXMOD,
                "psk_gemv_tc: bad args (K %% 64 == 0, 1..%d modules, workspace)", MAXMOD);
  PSK_CHECK_ARG(N > 0 && N % BN == 0, "psk_gemv_tc: N must be a positive multiple of %d", BN);
  const int maxm = max_rows_per_mod > 0 ? max_rows_per_mod : n_rows;
  if (n_rows == 0) return PSK_OK;
  cudaStream_t s = psk::as_stream(stream);
  if (maxm <= 16) return dispatch<16>(epilogue, x, n_rows, K, W_host, mod_row_start, n_mod, N, out, workspace, s);
  if (maxm <= 32) return dispatch<32>(epilogue, x, n_rows, K, W_host, mod_row_start, n_mod, N, out, workspace, s);
  if (maxm <= 64) return dispatch<64>(epilogue, x, n_rows, K, W_host, mod_row_start, n_mod, N, out, workspace, s);
  psk::set_error("psk_gemv_tc: more than 64 rows per module (%d)", maxm);
  return PSK_EINVAL;
}
