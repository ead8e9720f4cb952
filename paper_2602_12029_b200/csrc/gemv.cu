// K5 — grouped decode GEMV: y[r, n] = sum_k x[r, k] * W_mod(r)[n, k] for the
// 1..32 decode rows of each of n_mod co-batched decode modules.
//
// Decode is weight-streaming: every step reads each module's full weight
// set once (4 x 15 GB at the 8B shape) while the activation side is a few
// rows. The kernel is therefore built around keeping HBM saturated:
//
//   * persistent, one CTA per SM; the (module, weight-row) space is cut into
//     16-row tiles and each CTA owns a contiguous run of tiles (balanced to
//     within one tile; tiles never straddle modules since N % 16 == 0);
//   * warp 8 is a producer that streams each tile as 2048-column stages
//     (16 rows x 4 KiB) with cp.async.bulk (TMA bulk copies, L2 evict-first)
//     into a 3-stage shared-memory ring (~195 KiB in flight per SM) — it
//     does not wait on the previous kernel (PDL), so the first stages land
//     while that kernel drains. Measured on B200 (tools/bw_probe.cu): 4 KiB
//     row pieces stream at 6.95 TB/s, 2 KiB pieces at 5.74 TB/s;
//   * warps 0-7 each own 256 columns of every stage and run mma.sync
//     m16n8k16 (weights = A, 16 rows; activations = B, 8 rows per n-tile)
//     with a fixed k-permutation inside every 32-column group (applied to W
//     and x alike: a dot product is order-invariant) so every fragment is
//     one 16-byte shared-memory read (rows padded by 64 B: conflict-free);
//     x fragments come from L2 (ncu: re-reading them per tile cost 1.3 GB
//     of L2 traffic per gate/up launch at 8 rows/module; per group: 1/TG);
//   * tiles are walked in groups of up to TG (7 / 3 / 1 for <= 8 / 16 / 32
//     rows per module) with the K chunks outer: x fragments are loaded once
//     per (group, chunk) and reused for every tile of the group, the group's
//     accumulators stay in registers, and at the end of a group the 8 warps'
//     partials meet in shared memory and are summed in a fixed order —
//     results are bit-reproducible — then the fused epilogue
//     stores bf16 / fp32, adds into the fp32 residual stream, or applies
//     SiLU(gate)*up: gate/up rows are interleaved in 8-row groups, so each
//     16-row tile holds 8 gate + 8 matching up rows.
//
// Replaces the per-module dense projections of the reference decode forward
// (frontend/src/model.ts:298-306 q/k/v, :318 o-proj, :322-323 MLP, :334
// logits), executed here for all decode modules of a step in one launch.
#include "common.cuh"
#include "mma.cuh"
#include "tma.cuh"

namespace psk {
namespace gemv {

constexpr int CW = 8;                      // consumer warps
constexpr int THREADS = (CW + 1) * 32;     // + one producer warp
constexpr int TR = 16;                     // weight rows per tile (MMA M)
constexpr int WC = 256;                    // columns per consumer warp per stage
constexpr int GR = WC / 32;                // 32-column groups per warp per stage
constexpr int KC = CW * WC;                // columns per stage
constexpr int ROW_BYTES = KC * 2 + 64;     // padded shared-memory row
constexpr int STAGE_BYTES = TR * ROW_BYTES;
constexpr int SMEM_LIMIT = 227 * 1024;

template <int NT>
struct Cfg {
  static constexpr int MAXM = NT * 8;  // activation rows per module
  static constexpr int STAGES = 3;
  // tiles per group: their accumulators stay in registers across the K
  // chunks and meet once in `red` [CW][TG*TR][MAXM] for the cross-warp sum
  static constexpr int TG = (SMEM_LIMIT - STAGES * STAGE_BYTES - 256) / (CW * TR * MAXM * 4);
  static constexpr int RED_BYTES = CW * TG * TR * MAXM * 4;
  static constexpr int SMEM = STAGES * STAGE_BYTES + RED_BYTES + 256;
  static_assert(TG >= 1 && SMEM <= SMEM_LIMIT, "shared memory budget");
};

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// 1-D TMA bulk copy global -> shared completing on `bar` (bytes % 16 == 0).
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
      "[%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(tma::sa(bar)), "l"(policy)
      : "memory");
}

__device__ __forceinline__ uint4 lds128(const unsigned char* p) {
  return *reinterpret_cast<const uint4*>(p);
}

// x fragments (B operand) of one stage for this thread: row nt*8+gq of the
// tile's module, columns [8tq, 8tq+8) of each of the warp's 32-column
// groups; zero outside the module's rows or past K.
template <int NT>
__device__ __forceinline__ void load_x(uint4 (&xf)[NT][GR], const __nv_bfloat16* __restrict__ X, int K,
                                       int xb, int M, int c, int warp, int gq, int tq) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int row = nt * 8 + gq;
#pragma unroll
    for (int g = 0; g < GR; ++g) {
      const int col = c * KC + warp * WC + g * 32 + tq * 8;
      xf[nt][g] = (row < M && col < K)
                      ? __ldg(reinterpret_cast<const uint4*>(X + (int64_t)(xb + row) * K + col))
                      : make_uint4(0, 0, 0, 0);
    }
  }
}

// Walk order of one CTA: its tiles are cut into groups of <= TG consecutive
// tiles of one module; per group the K chunks are the outer loop, so each
// warp loads its x fragments of a chunk once and reuses them for every tile
// of the group (x is re-read from L2 once per group, not once per tile).
__device__ __forceinline__ int group_end(int gt0, int t1, int tg, int tpm) {
  return min(min(gt0 + tg, t1), (gt0 / tpm + 1) * tpm);
}

template <int NT, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
    gemv_kernel(const __nv_bfloat16* __restrict__ X, int K, const __nv_bfloat16* const* __restrict__ W,
                const int32_t* __restrict__ mrs, int n_mod, int N, void* __restrict__ out) {
  using C = Cfg<NT>;
  constexpr int MAXM = C::MAXM, TG = C::TG;
  extern __shared__ __align__(128) unsigned char smem[];
  float* red = reinterpret_cast<float*>(smem + C::STAGES * STAGE_BYTES);  // [CW][TG*TR][MAXM]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::STAGES * STAGE_BYTES + C::RED_BYTES);
  uint64_t* empty = full + C::STAGES;

  const int tpm = N / TR;  // tiles per module
  const int tiles = n_mod * tpm;
  const int t0 = (int)((int64_t)blockIdx.x * tiles / gridDim.x);
  const int t1 = (int)((int64_t)(blockIdx.x + 1) * tiles / gridDim.x);
  const int cpt = (K + KC - 1) / KC;  // K chunks (stages) per tile
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      tma::mbar_init(&full[s], 1);
      tma::mbar_init(&empty[s], CW);
    }
    tma::fence_mbar_init();
  }
  __syncthreads();
  pdl_trigger();

  if (warp == CW) {
    // ---- producer: weights do not depend on the previous kernel ----
    const uint64_t pol = policy_evict_first();
    int j = 0;
    for (int gt0 = t0; gt0 < t1;) {
      const int gt1 = group_end(gt0, t1, TG, tpm);
      const int mod = gt0 / tpm;
      const bool live = mrs[mod + 1] > mrs[mod];  // module without rows this step: no loads
      for (int c = 0; c < cpt; ++c) {
        const int cols = min(KC, K - c * KC);
        for (int t = gt0; t < gt1; ++t, ++j) {
          const int s = j % C::STAGES;
          tma::mbar_wait(&empty[s], ((j / C::STAGES) & 1) ^ 1);
          if (!live) {
            if (lane == 0) tma::mbar_arrive(&full[s]);
            continue;
          }
          if (lane == 0) tma::mbar_expect_tx(&full[s], TR * cols * 2);
          __syncwarp();
          if (lane < TR) {
            const __nv_bfloat16* src = W[mod] + ((int64_t)(t % tpm) * TR + lane) * K + (int64_t)c * KC;
            bulk_g2s(tma::sa(smem + s * STAGE_BYTES + lane * ROW_BYTES), src, cols * 2, &full[s], pol);
          }
        }
      }
      gt0 = gt1;
    }
    return;
  }

  // ---- consumers ----
  const int gq = lane >> 2, tq = lane & 3;
  pdl_wait();  // x (and the residual stream) come from the previous kernel
  int j = 0;
  for (int gt0 = t0; gt0 < t1;) {
    const int gt1 = group_end(gt0, t1, TG, tpm);
    const int ng = gt1 - gt0;
    const int mod = gt0 / tpm;
    const int xb = mrs[mod], M = mrs[mod + 1] - xb;
    float acc[TG][NT][4];
#pragma unroll
    for (int i = 0; i < TG; ++i)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) acc[i][nt][0] = acc[i][nt][1] = acc[i][nt][2] = acc[i][nt][3] = 0.f;
    for (int c = 0; c < cpt; ++c) {
      uint4 xc[NT][GR];
      load_x<NT>(xc, X, K, xb, M, c, warp, gq, tq);  // once per (group, chunk)
#pragma unroll
      for (int i = 0; i < TG; ++i) {
        if (i >= ng) break;
        const int s = j % C::STAGES;
        tma::mbar_wait(&full[s], (j / C::STAGES) & 1);
        if (M > 0) {
          const unsigned char* st = smem + s * STAGE_BYTES + (warp * WC + tq * 8) * 2;
#pragma unroll
          for (int g = 0; g < GR; ++g) {
            const bool ok = c * KC + warp * WC + g * 32 + tq * 8 < K;
            const uint4 wa = ok ? lds128(st + gq * ROW_BYTES + g * 64) : make_uint4(0, 0, 0, 0);
            const uint4 wb = ok ? lds128(st + (gq + 8) * ROW_BYTES + g * 64) : make_uint4(0, 0, 0, 0);
            const uint32_t a0[4] = {wa.x, wb.x, wa.y, wb.y};
            const uint32_t a1[4] = {wa.z, wb.z, wa.w, wb.w};
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) {
              if (nt * 8 >= M) break;
              mma_bf16_16816(acc[i][nt], a0, xc[nt][g].x, xc[nt][g].y);
              mma_bf16_16816(acc[i][nt], a1, xc[nt][g].z, xc[nt][g].w);
            }
          }
        }
        __syncwarp();
        if (lane == 0) tma::mbar_arrive(&empty[s]);
        ++j;
      }
    }

    // ---- group complete: reduce the 8 warps' partials, fused epilogue ----
    if (M > 0) {
      float* mine = red + warp * TG * TR * MAXM;
#pragma unroll
      for (int i = 0; i < TG; ++i) {
        if (i >= ng) break;
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const int m = nt * 8 + 2 * tq;
          float* r0 = mine + (i * TR + gq) * MAXM + m;
          float* r8 = r0 + 8 * MAXM;
          r0[0] = acc[i][nt][0];
          r0[1] = acc[i][nt][1];
          r8[0] = acc[i][nt][2];
          r8[1] = acc[i][nt][3];
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");
    if (M > 0) {
      const int n0 = (gt0 % tpm) * TR;  // first weight row of the group in its module
      if (EPI == PSK_EPI_SILU_MUL) {
        // tile = [gate 8 | up 8] rows -> 8 outputs
        for (int e = threadIdx.x; e < ng * 8 * M; e += CW * 32) {
          const int m = e / (ng * 8), q = e % (ng * 8);
          const int i = q >> 3, r = q & 7;
          float gv = 0.f, uv = 0.f;
#pragma unroll
          for (int w = 0; w < CW; ++w) {
            const float* rw = red + ((w * TG + i) * TR + r) * MAXM + m;
            gv += rw[0];
            uv += rw[8 * MAXM];
          }
          const float sg = gv / (1.f + __expf(-gv));
          reinterpret_cast<__nv_bfloat16*>(out)[(int64_t)(xb + m) * (N / 2) + n0 / 2 + q] = f2bf(sg * uv);
        }
      } else {
        for (int e = threadIdx.x; e < ng * TR * M; e += CW * 32) {
          const int m = e / (ng * TR), q = e % (ng * TR);  // q = row within the group
          float v = 0.f;
#pragma unroll
          for (int w = 0; w < CW; ++w) v += red[((w * TG) * TR + q) * MAXM + m];
          const int64_t o = (int64_t)(xb + m) * N + n0 + q;
          if (EPI == PSK_EPI_STORE_BF16) reinterpret_cast<__nv_bfloat16*>(out)[o] = f2bf(v);
          if (EPI == PSK_EPI_STORE_F32) reinterpret_cast<float*>(out)[o] = v;
          if (EPI == PSK_EPI_RESID_ADD) reinterpret_cast<float*>(out)[o] += v;
        }
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(CW * 32) : "memory");  // red is rewritten by the next group
    gt0 = gt1;
  }
}

template <int NT, int EPI>
int launch(const void* x, int K, const void* const* W, const int32_t* mrs, int n_mod, int N, void* out,
           cudaStream_t s) {
  static bool attr_set = false;
  auto k = gemv_kernel<NT, EPI>;
  if (!attr_set) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<NT>::SMEM));
    attr_set = true;
  }
  const int sms = psk::sm_budget();
  const int tiles = n_mod * (N / TR);
  const int grid = tiles < sms ? tiles : sms;
  PSK_CUDA_TRY(psk::launch_pdl(k, dim3(grid), dim3(THREADS), (size_t)Cfg<NT>::SMEM, s,
                               reinterpret_cast<const __nv_bfloat16*>(x), K,
                               reinterpret_cast<const __nv_bfloat16* const*>(W), mrs, n_mod, N, out));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

template <int NT>
int dispatch(int epi, const void* x, int K, const void* const* W, const int32_t* mrs, int n_mod, int N,
             void* out, cudaStream_t s) {
  switch (epi) {
    case PSK_EPI_STORE_BF16: return launch<NT, PSK_EPI_STORE_BF16>(x, K, W, mrs, n_mod, N, out, s);
    case PSK_EPI_STORE_F32: return launch<NT, PSK_EPI_STORE_F32>(x, K, W, mrs, n_mod, N, out, s);
    case PSK_EPI_RESID_ADD: return launch<NT, PSK_EPI_RESID_ADD>(x, K, W, mrs, n_mod, N, out, s);
    case PSK_EPI_SILU_MUL: return launch<NT, PSK_EPI_SILU_MUL>(x, K, W, mrs, n_mod, N, out, s);
  }
  psk::set_error("psk_gemv: unknown epilogue %d", epi);
  return PSK_EINVAL;
}

}  // namespace gemv
}  // namespace psk

extern "C" int psk_gemv(const void* x, int32_t n_rows, int32_t K, const void* const* W,
                        const int32_t* mod_row_start, int32_t n_mod, int32_t max_rows_per_mod, int32_t N,
                        int32_t epilogue, void* out, void* stream) {
  PSK_CHECK_ARG(x && W && mod_row_start && out && n_rows >= 0 && K > 0 && K % 8 == 0 && n_mod > 0,
                "psk_gemv: bad args (K must be a positive multiple of 8)");
  PSK_CHECK_ARG(N > 0 && N % 16 == 0, "psk_gemv: N must be a positive multiple of 16");
  const int maxm = max_rows_per_mod > 0 ? max_rows_per_mod : n_rows;
  if (n_rows == 0) return PSK_OK;
  cudaStream_t s = psk::as_stream(stream);
  using namespace psk::gemv;
  if (maxm <= 8) return dispatch<1>(epilogue, x, K, W, mod_row_start, n_mod, N, out, s);
  if (maxm <= 16) return dispatch<2>(epilogue, x, K, W, mod_row_start, n_mod, N, out, s);
  if (maxm <= 32) return dispatch<4>(epilogue, x, K, W, mod_row_start, n_mod, N, out, s);
  psk::set_error("psk_gemv: more than 32 rows per module (%d)", maxm);
  return PSK_EINVAL;
}
