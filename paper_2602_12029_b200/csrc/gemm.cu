// K1 + K2 — prefill GEMMs on the 5th-gen tensor cores.
//
// C[M,N] = A[M,K] . B[N,K]^T, bf16 operands (both K-major), fp32 accumulate
// in TMEM. Replaces the dense contractions of the reference forward
// (frontend/src/model.ts:298-306 q/k/v, :318 o-proj, :322-323 MLP) which the
// simulator only models as time (src/prefillsim/costs.py:46-54).
//
// Kernel anatomy (persistent, one CTA per SM, 8 warps):
//   warp 0     TMA producer: 128x64 A and 256x64 B boxes, 128B-swizzled,
//              into a 4-stage shared-memory ring (48 KiB / stage)
//   warp 1     MMA issuer: one elected lane issues tcgen05.mma (M=128,
//              N=256, K=16) x4 per stage; tcgen05.commit frees the stage
//   warp 2     TMEM allocator (512 columns = two 128x256 fp32 accumulators)
//   warps 4-7  epilogue: tcgen05.ld 32x32b.x32 (thread = tile row), fused
//              epilogue, stores; accumulator stage released via mbarrier so
//              the MMA of tile i+1 overlaps the epilogue of tile i.
// Tiles are walked m-fastest so one wave shares its B (weight) tiles in L2.
// Default kernel: the CTA-pair variant below (gemm_pair_kernel, 256x256
// tiles on two SMs with tcgen05 cta_group::2, half of B staged per SM);
// PSK_GEMM_PAIR=0 selects this 1-SM kernel, which also remains the split-K
// path when a workspace is bound.
//
// Fused epilogues: bf16 store, fp32 residual add, SiLU(gate)*up over the
// [gate8|up8]-interleaved weight layout, and QKV -> RoPE (rotate-half) ->
// q_rot + paged K/V write (K2, model.ts:307-311 cache push, done in place).
#include "common.cuh"

#include <cuda.h>

namespace psk {
namespace gemm {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int THREADS = 256;
constexpr int TMEM_COLS = 512;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

struct Epi {
  int mode;
  void* out;
  int64_t ldo;
  // QKV_ROPE_KV
  const float* rope;
  int pos0;
  int nq, nkv;
  psk_kv_layout kv;
  int layer;
  const int32_t* page_table;
  __nv_bfloat16* q_out;
  // batched (varlen) prefill: per-row absolute position and KV slot
  // (page * 16 + token in page); nullptr = one sequence at pos0 + row
  const int32_t* row_pos;
  const int32_t* row_slot;
};

// ----------------------------------------------------------- PTX helpers --

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_addr(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(a),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x,
                                            int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(smem_addr(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  // K-major, 128B swizzle: LBO = 16 B (unused), SBO = 1024 B (8 rows x 128 B),
  // version 1 (sm100), layout SWIZZLE_128B (2) in bits 61-63.
  uint64_t d = (uint64_t)((smem_addr(p) >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// kind::f16 instruction descriptor: D fp32, A/B bf16, both K-major.
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_addr(bar))
               : "memory");
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float* v) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]),
      "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]),
      "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]),
      "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
      : "memory");
}

// ------------------------------------------------------------- epilogues --

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) reinterpret_cast<uint4*>(dst)[i] = f32_to_bf16x8(v + 8 * i);
}

__device__ __forceinline__ __nv_bfloat16* kv_dst(const psk_kv_layout& kv, int page, int layer,
                                                 int kvsel, int head, int tok) {
  return reinterpret_cast<__nv_bfloat16*>(kv.base) + (int64_t)page * kv.page_elems +
         ((((int64_t)layer * 2 + kvsel) * kv.n_kv_heads + head) * kv.page_tokens + tok) * kv.head_dim;
}

// Epilogue for one 128x256 tile; thread owns tile row `r` (TMEM lane).
__device__ void epilogue_tile(const Epi& e, uint32_t tacc, int row, bool row_ok, int n0, int ncols = BN) {
  float v[32], w[32];
  if (e.mode == PSK_EPI_QKV_ROPE_KV) {
    int pos = e.pos0 + row, page = 0, tok = 0;
    if (row_ok) {
      if (e.row_pos != nullptr) {
        pos = e.row_pos[row];
        const int slot = e.row_slot[row];
        page = slot >> 4;
        tok = slot & 15;
      } else {
        page = e.page_table[pos / 16];
        tok = pos % 16;
      }
    }
    const float* cs = e.rope + (int64_t)pos * 128;
#pragma unroll 1
    for (int hh = 0; hh < ncols / 128; ++hh) {
      const int head = (n0 >> 7) + hh;
      const uint32_t hb = tacc + hh * 128;
      if (head >= e.nq + e.nkv) {  // V head: plain copy into the page
        const int vh = head - e.nq - e.nkv;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          tmem_ld32(hb + c * 32, v);
          if (row_ok) store_bf16x32(kv_dst(e.kv, page, e.layer, 1, vh, tok) + c * 32, v);
        }
        continue;
      }
#pragma unroll 1
      for (int half = 0; half < 2; ++half) {
        tmem_ld32(hb + half * 32, v);       // dims [32h, 32h+32)
        tmem_ld32(hb + half * 32 + 64, w);  // dims [64+32h, ...)
        if (!row_ok) continue;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float c = cs[2 * (half * 32 + j)], s = cs[2 * (half * 32 + j) + 1];
          const float x1 = v[j], x2 = w[j];
          v[j] = x1 * c - x2 * s;
          w[j] = x2 * c + x1 * s;
        }
        __nv_bfloat16* dst;
        if (head < e.nq) {
          dst = e.q_out + ((int64_t)row * e.nq + head) * 128;
        } else {
          dst = kv_dst(e.kv, page, e.layer, 0, head - e.nq, tok);
        }
        store_bf16x32(dst + half * 32, v);
        store_bf16x32(dst + half * 32 + 64, w);
      }
    }
    return;
  }
#pragma unroll 1
  for (int c = 0; c < ncols / 32; ++c) {
    tmem_ld32(tacc + c * 32, v);
    if (!row_ok) continue;
    const int col = n0 + c * 32;
    if (e.mode == PSK_EPI_STORE_BF16) {
      store_bf16x32(reinterpret_cast<__nv_bfloat16*>(e.out) + (int64_t)row * e.ldo + col, v);
    } else if (e.mode == PSK_EPI_STORE_F32) {
      float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (int64_t)row * e.ldo + col);
#pragma unroll
      for (int i = 0; i < 8; ++i) d[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    } else if (e.mode == PSK_EPI_RESID_ADD) {
      float4* d = reinterpret_cast<float4*>(reinterpret_cast<float*>(e.out) + (int64_t)row * e.ldo + col);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 o = d[i];
        o.x += v[4 * i];
        o.y += v[4 * i + 1];
        o.z += v[4 * i + 2];
        o.w += v[4 * i + 3];
        d[i] = o;
      }
    } else if (e.mode == PSK_EPI_SILU_MUL) {
      // 32 columns = [gate 8 | up 8 | gate 8 | up 8] -> 16 outputs
      float o[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int b = (i >> 3) * 16 + (i & 7);
        const float g = v[b], u = v[b + 8];
        o[i] = g / (1.f + __expf(-g)) * u;
      }
      __nv_bfloat16* d = reinterpret_cast<__nv_bfloat16*>(e.out) + (int64_t)row * e.ldo + col / 2;
      reinterpret_cast<uint4*>(d)[0] = f32_to_bf16x8(o);
      reinterpret_cast<uint4*>(d)[1] = f32_to_bf16x8(o + 8);
    }
  }
}

// ---------------------------------------------------------------- kernel --

// Work schedule. Tiles are walked m-fastest, item = blockIdx.x + i * grid.
// When the last wave would be mostly idle (tiles = W * grid + rem with
// rem <= grid / 2), the `rem` tail tiles are split along K into S pieces
// (S = grid / rem, >= 4 k-blocks each) so the tail costs 1/S of a tile
// instead of a whole one (4096^2 GEMMs: 512 tiles = 3.46 waves -> 3.5, not 4).
// Each split writes its fp32 partial to the workspace; the last one to
// finish (atomic counter) sums all S partials in split order (fixed order:
// bit-reproducible), stores the sum back into its TMEM accumulator and runs
// the normal fused epilogue. That reduction (one CTA re-reading S x 128 KiB)
// measured slower end to end, so by default (no workspace bound) the tail
// tiles are split along N instead: S independent 128 x (256 / S) pieces
// (MMA N = 256 / S, B box of 256 / S rows, the epilogue on those columns),
// no reduction at all (S <= 2 for the QKV/RoPE epilogue: whole heads).
struct Sched {
  int tiles, full, rem, S, items;
  int split_n;     // 1: tail pieces along N; 0: along K (workspace)
  float* part;     // [rem * S][BM][BN] fp32
  int* counters;   // [rem], zero between launches
};

__device__ __forceinline__ void item_range(const Sched& sc, int item, int kb_n, int& tile, int& kb0, int& kb1,
                                           int& split, int& piece) {
  piece = -1;
  split = -1;
  kb0 = 0;
  kb1 = kb_n;
  if (item < sc.full) {
    tile = item;
  } else {
    const int j = item - sc.full;
    tile = sc.full + j / sc.S;
    if (sc.split_n) {
      piece = j % sc.S;
    } else {
      split = j % sc.S;
      kb0 = split * kb_n / sc.S;
      kb1 = (split + 1) * kb_n / sc.S;
    }
  }
}

// Tile order: m-fastest inside groups of GROUP_ROWS rows, group by group.
// Inside a group a wave shares its weight (B) tiles in L2 and the group's A
// rows (4096 x K bf16 <= 117 MiB at K = 14336, 33.5 MiB at K = 4096) stay
// L2-resident while every n column passes over them; plain m-fastest order
// over a taller A re-streams all of A from HBM once per n column.
constexpr int GROUP_ROWS = 4096;

__device__ __forceinline__ void tile_coords(int t, int m_tiles, int n_tiles, int gm, int& mb, int& nb) {
  const int g = t / (gm * n_tiles);
  const int m0 = g * gm;
  const int rows = m_tiles - m0 < gm ? m_tiles - m0 : gm;
  const int r = t - g * gm * n_tiles;
  mb = m0 + r % rows;
  nb = r / rows;
}

__global__ void __launch_bounds__(THREADS, 1)
    gemm_bf16_tn_kernel(const __grid_constant__ CUtensorMap tmap_a,
                        const __grid_constant__ CUtensorMap tmap_b, const __grid_constant__ CUtensorMap tmap_bp,
                        int M, int N, int K, Epi e, Sched sc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tiles = (M + BM - 1) / BM;
  const int kb_n = K / BK;
  __shared__ int s_last;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmap_a);
    tma_prefetch(&tmap_b);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_addr(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: let the next kernel's CTAs start their prologue as SMs free up; the
  // activations (A, the residual, KV pages) are read only after the wait
  pdl_trigger();

  if (warp == 0) {
    if (lane == 0) {
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int item = blockIdx.x; item < sc.items; item += gridDim.x) {
        int t, kb0, kb1, split, piece;
        item_range(sc, item, kb_n, t, kb0, kb1, split, piece);
        int mb, nb;
        tile_coords(t, m_tiles, N / BN, GROUP_ROWS / BM, mb, nb);
        const int pn = BN / sc.S;  // N-piece width
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (piece >= 0) {  // tail piece: A tile + a (256 / S)-row B box
            mbar_expect_tx(&full[stage], A_BYTES + pn * BK * 2);
            tma_load_2d(&tmap_a, &full[stage], sA + stage * A_BYTES, kb * BK, mb * BM);
            tma_load_2d(&tmap_bp, &full[stage], sB + stage * B_BYTES, kb * BK, nb * BN + piece * pn);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(&tmap_a, &full[stage], sA + stage * A_BYTES, kb * BK, mb * BM);
          tma_load_2d(&tmap_b, &full[stage], sB + stage * B_BYTES, kb * BK, nb * BN);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_full = idesc_bf16(BM, BN);
      const uint32_t idesc_piece = idesc_bf16(BM, BN / (sc.S > 0 ? sc.S : 1));
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = blockIdx.x; item < sc.items; item += gridDim.x, ++it) {
        int t, kb0, kb1, split, piece;
        item_range(sc, item, kb_n, t, kb0, kb1, split, piece);
        const uint32_t idesc = piece >= 0 ? idesc_piece : idesc_full;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = smem_desc_sw128(sA + stage * A_BYTES);
          const uint64_t db = smem_desc_sw128(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            // +32 bytes along K inside the 128B swizzle atom = +2 in the
            // descriptor's 16-byte address units
            umma_bf16(tacc, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          }
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else if (warp >= 4) {
    pdl_wait();
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int r_in_tile = q * 32 + lane;
    int it = 0;
    for (int item = blockIdx.x; item < sc.items; item += gridDim.x, ++it) {
      int t, kb0, kb1, split, piece;
      item_range(sc, item, kb_n, t, kb0, kb1, split, piece);
      int mb, nb;
      tile_coords(t, m_tiles, N / BN, GROUP_ROWS / BM, mb, nb);
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = mb * BM + r_in_tile;
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (split >= 0) {
        // split-K tail tile: publish this split's partial; the last split
        // sums all partials (split order) into its accumulator
        const int ti = t - sc.full;
        float* mine = sc.part + ((int64_t)(ti * sc.S + split) * BM + r_in_tile) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
          tmem_ld32(tacc + c * 32, v);
#pragma unroll
          for (int i = 0; i < 8; ++i)
            reinterpret_cast<float4*>(mine + c * 32)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (warp == 4 && lane == 0) {
          const int old = atomicAdd(&sc.counters[ti], 1);
          s_last = old == sc.S - 1;
          if (s_last) {
            sc.counters[ti] = 0;  // ready for the next launch
            __threadfence();
          }
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (!s_last) {
          tc_fence_before();
          mbar_arrive(&tempty[acc]);
          continue;
        }
        const float* rows0 = sc.part + ((int64_t)(ti * sc.S) * BM + r_in_tile) * BN;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
          float v[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
          for (int sp = 0; sp < sc.S; ++sp) {
            const float4* src = reinterpret_cast<const float4*>(rows0 + (int64_t)sp * BM * BN + c * 32);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 x = __ldcg(src + i);
              v[4 * i] += x.x;
              v[4 * i + 1] += x.y;
              v[4 * i + 2] += x.z;
              v[4 * i + 3] += x.w;
            }
          }
          tmem_st32(tacc + c * 32, v);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (piece >= 0)
        epilogue_tile(e, tacc, row, row < M, nb * BN + piece * (BN / sc.S), BN / sc.S);
      else
        epilogue_tile(e, tacc, row, row < M, nb * BN);
      tc_fence_before();
      mbar_arrive(&tempty[acc]);
    }
  }
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ------------------------------------------------ CTA-pair (2-SM) variant --
//
// One cluster of two CTAs on a TPC computes a 256x256 tile with
// tcgen05.mma.cta_group::2 (M = 256: each CTA's TMEM holds its own 128 rows
// x 256 fp32 columns). Each CTA stages its 128 A rows and HALF of the B tile
// (128 of the 256 weight rows); the pair's tensor cores read the other half
// across the TPC, so per SM a k-block moves 32 KiB of operands through
// shared memory / L2 instead of 48 KiB (the 1-SM kernel's limit: 148 SMs x
// 48 KiB per 512-cycle k-block is above what L2 delivers). Only the leader
// (rank 0) issues MMAs; both CTAs' TMA loads complete on the leader's `full`
// barrier; the leader's commits multicast `empty` / `tfull` to both CTAs;
// both epilogues release the accumulator on the leader's `tempty` (256
// arrivals). Tail tiles split along N (pieces of 256 / S columns, MMA N =
// 256 / S, each CTA loads 128 / S weight rows) exactly like the 1-SM kernel.
namespace pair {

constexpr int BM2 = 256;                     // pair tile rows (128 per CTA)
constexpr int A_BYTES = BM * BK * 2;         // per CTA: 128 x 64
constexpr int B_BYTES = (BN / 2) * BK * 2;   // per CTA: 128 x 64 (half of B)
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int STAGES = 6;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t peer_addr(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_addr(local)), "r"(rank));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// TMA load whose completion (complete_tx) lands on the LEADER CTA's barrier:
// the barrier's shared::cta address with the peer bit (24) cleared.
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(smem_addr(dst)),
      "l"(map), "r"(smem_addr(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void umma2_bf16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}

// arrive (once, when this thread's prior MMAs complete) on `bar` in both CTAs
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_addr(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// Warp-converged forms (the whole warp executes them with warp-uniform
// operands, one elected lane issues; from an if (lane == 0) branch each TMA /
// MMA became an R2UR.BROADCAST waterfall loop).
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(
          smem_addr(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_pair_e(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];\n}\n" ::"r"(smem_addr(dst)),
      "l"(map), "r"(smem_addr(bar) & 0xFEFFFFFFu), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma2_bf16_e(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n.reg .pred p, e;\nelect.sync _|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma2_commit_both_e(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_addr(bar)),
      "h"((uint16_t)3)
      : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmap_a, const __grid_constant__ CUtensorMap tmap_b,
                     const __grid_constant__ CUtensorMap tmap_bp, int M, int N, int K, Epi e, Sched sc) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  unsigned char* sA = smem;
  unsigned char* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  const int m_tiles = (M + BM2 - 1) / BM2;
  const int kb_n = K / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmap_a);
    tma_prefetch(&tmap_b);
    tma_prefetch(&tmap_bp);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 256);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // PDL: let the next kernel's CTAs start their prologue as SMs free up; the
  // activations (A, the residual, KV pages) are read only after the wait
  pdl_trigger();

  if (warp == 0) {
    {
      pdl_wait();
      int stage = 0;
      uint32_t phase = 0;
      for (int item = pair; item < sc.items; item += n_pairs) {
        int t, kb0, kb1, split, piece;
        item_range(sc, item, kb_n, t, kb0, kb1, split, piece);
        int mb, nb;
        tile_coords(t, m_tiles, N / BN, GROUP_ROWS / BM2, mb, nb);
        const int row0 = mb * BM2 + (int)rank * BM;
        const int hp = BN / sc.S / 2;  // this CTA's share of a tail piece's weight rows
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (piece >= 0) {
            if (rank == 0) mbar_expect_tx_e(&full[stage], 2 * (A_BYTES + hp * BK * 2));
            tma_load_2d_pair_e(&tmap_a, &full[stage], sA + stage * A_BYTES, kb * BK, row0);
            tma_load_2d_pair_e(&tmap_bp, &full[stage], sB + stage * B_BYTES, kb * BK,
                             nb * BN + piece * 2 * hp + (int)rank * hp);
          } else {
            if (rank == 0) mbar_expect_tx_e(&full[stage], 2 * STAGE_BYTES);
            tma_load_2d_pair_e(&tmap_a, &full[stage], sA + stage * A_BYTES, kb * BK, row0);
            tma_load_2d_pair_e(&tmap_b, &full[stage], sB + stage * B_BYTES, kb * BK, nb * BN + (int)rank * (BN / 2));
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (rank == 0) {
      constexpr uint32_t idesc_full = idesc_bf16(BM2, BN);
      const uint32_t idesc_piece = idesc_bf16(BM2, BN / sc.S);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int item = pair; item < sc.items; item += n_pairs, ++it) {
        int t, kb0, kb1, split, piece;
        item_range(sc, item, kb_n, t, kb0, kb1, split, piece);
        const uint32_t idesc = piece >= 0 ? idesc_piece : idesc_full;
        const int acc = it & 1;
        mbar_wait(&tempty[acc], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t tacc = tmem_base + acc * BN;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = smem_desc_sw128(sA + stage * A_BYTES);
          const uint64_t db = smem_desc_sw128(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma2_bf16_e(tacc, da + 2 * k, db + 2 * k, idesc, (kb != kb0 || k != 0) ? 1u : 0u);
          umma2_commit_both_e(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma2_commit_both_e(&tfull[acc]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    pdl_wait();
    const int q = warp & 3;
    const int r_in_tile = q * 32 + lane;
    const uint32_t tempty_leader = peer_addr(tempty, 0);
    int it = 0;
    for (int item = pair; item < sc.items; item += n_pairs, ++it) {
      int t, kb0, kb1, split, piece;
      item_range(sc, item, kb_n, t, kb0, kb1, split, piece);
      int mb, nb;
      tile_coords(t, m_tiles, N / BN, GROUP_ROWS / BM2, mb, nb);
      const int acc = it & 1;
      mbar_wait(&tfull[acc], (it >> 1) & 1);
      tc_fence_after();
      const int row = mb * BM2 + (int)rank * BM + r_in_tile;
      const uint32_t tacc = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (piece >= 0)
        epilogue_tile(e, tacc, row, row < M, nb * BN + piece * (BN / sc.S), BN / sc.S);
      else
        epilogue_tile(e, tacc, row, row < M, nb * BN);
      tc_fence_before();
      asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_leader + acc * 8)
                   : "memory");
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

}  // namespace pair

// ------------------------------------------------------------ host side --

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

static int make_map(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int box_rows) {
  EncodeTiledFn enc = get_encode();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return PSK_ECUDA;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                   es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return PSK_ECUDA;
  }
  return PSK_OK;
}

// split-K workspace (psk_gemm_bind_workspace); none bound = no split
struct Workspace {
  float* part = nullptr;
  int64_t part_bytes = 0;
  int* counters = nullptr;
  int n_counters = 0;
};
static Workspace g_ws;
constexpr int64_t WS_COUNTER_BYTES = 4096;

// CTA-pair kernel unless PSK_GEMM_PAIR=0 (1-SM kernel, kept for A/B runs
// and as the split-K path when a workspace is bound).
static bool use_pair() {
  static int v = -1;
  if (v < 0) {
    const char* env = getenv("PSK_GEMM_PAIR");
    v = (env && env[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

static int launch_pair(const CUtensorMap& ma, const void* B, int M, int N, int K, const Epi& e, cudaStream_t s,
                       int sms) {
  static bool attr = false;
  if (!attr) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(pair::gemm_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      pair::SMEM_BYTES));
    attr = true;
  }
  CUtensorMap mb, mbp;
  int rc = make_map(&mb, B, N, K, BN / 2);
  if (rc) return rc;
  const int tiles = ((M + pair::BM2 - 1) / pair::BM2) * (N / BN);
  const int max_pairs = sms / 2;
  const int pairs = tiles < max_pairs ? tiles : max_pairs;
  Sched sc{};
  sc.tiles = tiles;
  sc.full = tiles;
  sc.S = 1;
  sc.split_n = 1;
  mbp = mb;
  const int rem = tiles % pairs, waves = tiles / pairs;
  if (waves >= 1 && rem > 0 && rem <= pairs / 2) {
    // split-N tail pieces of 256 / S columns (QKV/RoPE: whole heads)
    int S = pairs / rem >= 4 ? 4 : 2;
    if (e.mode == PSK_EPI_QKV_ROPE_KV) S = 2;
    rc = make_map(&mbp, B, N, K, BN / S / 2);
    if (rc) return rc;
    sc.full = tiles - rem;
    sc.rem = rem;
    sc.S = S;
  }
  sc.items = sc.full + sc.rem * sc.S;
  PSK_CUDA_TRY(launch_pdl(pair::gemm_pair_kernel, dim3(2 * pairs), dim3(THREADS), (size_t)pair::SMEM_BYTES, s,
                          ma, mb, mbp, M, N, K, e, sc));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

static int launch(const void* A, const void* B, int M, int N, int K, const Epi& e, cudaStream_t s) {
  if (M <= 0) return PSK_OK;
  if (N % BN != 0 || K % BK != 0) {
    set_error("psk_gemm: N %% 256 and K %% 64 must be 0 (N=%d K=%d)", N, K);
    return PSK_EINVAL;
  }
  CUtensorMap ma, mb;
  int rc = make_map(&ma, A, M, K, BM);
  if (rc) return rc;
  rc = make_map(&mb, B, N, K, BN);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(gemm_bf16_tn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      SMEM_BYTES));
    attr = true;
  }
  const int sms = sm_budget();
  if (!g_ws.part && use_pair()) return launch_pair(ma, B, M, N, K, e, s, sms);
  const int tiles = ((M + BM - 1) / BM) * (N / BN);
  const int grid = tiles < sms ? tiles : sms;
  Sched sc{};
  sc.tiles = tiles;
  sc.full = tiles;
  sc.rem = 0;
  sc.S = 1;
  sc.split_n = 0;
  const int kb_n = K / BK;
  const int rem = tiles % grid, waves = tiles / grid;
  CUtensorMap mbp = mb;
  if (!g_ws.part && waves >= 1 && rem > 0 && rem <= grid / 2) {
    // split-N tail: S pieces of 256 / S columns (QKV/RoPE: whole 128-column heads)
    int S = grid / rem >= 4 ? 4 : 2;
    if (e.mode == PSK_EPI_QKV_ROPE_KV) S = 2;
    rc = make_map(&mbp, B, N, K, BN / S);
    if (rc) return rc;
    sc.full = tiles - rem;
    sc.rem = rem;
    sc.S = S;
    sc.split_n = 1;
  }
  if (g_ws.part && waves >= 1 && rem > 0 && rem <= grid / 2) {
    int S = grid / rem;
    if (S > kb_n / 4) S = kb_n / 4;
    if (S >= 2 && (int64_t)rem * S * BM * BN * 4 <= g_ws.part_bytes && rem <= g_ws.n_counters) {
      sc.full = tiles - rem;
      sc.rem = rem;
      sc.S = S;
      sc.part = g_ws.part;
      sc.counters = g_ws.counters;
    }
  }
  sc.items = sc.full + sc.rem * sc.S;
  PSK_CUDA_TRY(launch_pdl(gemm_bf16_tn_kernel, dim3(grid), dim3(THREADS), (size_t)SMEM_BYTES, s, ma, mb, mbp, M, N,
                          K, e, sc));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // namespace gemm
}  // namespace psk

extern "C" {

int psk_gemm_workspace(int64_t* bytes) {
  PSK_CHECK_ARG(bytes != nullptr, "psk_gemm_workspace: null out");
  const int sms = psk::device_sms();
  *bytes = psk::gemm::WS_COUNTER_BYTES + (int64_t)sms * psk::gemm::BM * psk::gemm::BN * 4;
  return PSK_OK;
}

int psk_gemm_bind_workspace(void* ws, int64_t bytes) {
  using namespace psk::gemm;
  if (ws == nullptr) {
    g_ws = Workspace{};
    return PSK_OK;
  }
  PSK_CHECK_ARG(bytes > WS_COUNTER_BYTES, "psk_gemm_bind_workspace: workspace too small");
  g_ws.counters = reinterpret_cast<int*>(ws);
  g_ws.n_counters = (int)(WS_COUNTER_BYTES / 4);
  g_ws.part = reinterpret_cast<float*>(reinterpret_cast<char*>(ws) + WS_COUNTER_BYTES);
  g_ws.part_bytes = bytes - WS_COUNTER_BYTES;
  return PSK_OK;
}

int psk_gemm(const void* A, const void* B, int32_t M, int32_t N, int32_t K, int32_t epilogue,
             void* out, int64_t ldo, void* stream) {
  PSK_CHECK_ARG(A && B && out && epilogue >= 0 && epilogue <= PSK_EPI_SILU_MUL,
                "psk_gemm: bad args");
  psk::gemm::Epi e{};
  e.mode = epilogue;
  e.out = out;
  e.ldo = ldo;
  return psk::gemm::launch(A, B, M, N, K, e, psk::as_stream(stream));
}

int psk_gemm_qkv_rope_kv(const void* A, const void* Wqkv, int32_t T, int32_t K, int32_t n_q_heads,
                         const float* rope, int32_t pos0, psk_kv_layout kv, int32_t layer,
                         const int32_t* page_table, void* q_out, void* stream) {
  PSK_CHECK_ARG(A && Wqkv && rope && page_table && q_out && kv.head_dim == 128 && kv.page_tokens == 16,
                "psk_gemm_qkv_rope_kv: bad args");
  psk::gemm::Epi e{};
  e.mode = PSK_EPI_QKV_ROPE_KV;
  e.rope = rope;
  e.pos0 = pos0;
  e.nq = n_q_heads;
  e.nkv = kv.n_kv_heads;
  e.kv = kv;
  e.layer = layer;
  e.page_table = page_table;
  e.q_out = reinterpret_cast<__nv_bfloat16*>(q_out);
  const int N = (n_q_heads + 2 * kv.n_kv_heads) * 128;
  return psk::gemm::launch(A, Wqkv, T, N, K, e, psk::as_stream(stream));
}

int psk_gemm_qkv_rope_kv_rows(const void* A, const void* Wqkv, int32_t T, int32_t K, int32_t n_q_heads,
                              const float* rope, const int32_t* row_pos, const int32_t* row_slot,
                              psk_kv_layout kv, int32_t layer, void* q_out, void* stream) {
  PSK_CHECK_ARG(A && Wqkv && rope && row_pos && row_slot && q_out && kv.head_dim == 128 && kv.page_tokens == 16,
                "psk_gemm_qkv_rope_kv_rows: bad args");
  psk::gemm::Epi e{};
  e.mode = PSK_EPI_QKV_ROPE_KV;
  e.rope = rope;
  e.nq = n_q_heads;
  e.nkv = kv.n_kv_heads;
  e.kv = kv;
  e.layer = layer;
  e.row_pos = row_pos;
  e.row_slot = row_slot;
  e.q_out = reinterpret_cast<__nv_bfloat16*>(q_out);
  const int N = (n_q_heads + 2 * kv.n_kv_heads) * 128;
  return psk::gemm::launch(A, Wqkv, T, N, K, e, psk::as_stream(stream));
}

}  // extern "C"
