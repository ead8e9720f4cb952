// mbarrier / TMA / cluster (DSMEM) PTX helpers shared by the sm_100a kernels.
#pragma once

#include <cuda.h>
#include <stdint.h>

namespace psk {
namespace tma {

__device__ __forceinline__ uint32_t sa(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(count));
}

__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(sa(bar)),
      "r"(parity)
      : "memory");
}

// 2D tiled TMA load (box given by the tensor map) completing on `bar`.
__device__ __forceinline__ void load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
      "%4}], [%2];" ::"r"(sa(dst)),
      "l"(map), "r"(sa(bar)), "r"(x), "r"(y)
      : "memory");
}

// 3D tiled TMA load (box given by the tensor map) completing on `bar`.
__device__ __forceinline__ void load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], "
      "[%2];" ::"r"(sa(dst)),
      "l"(map), "r"(sa(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// 4D tiled TMA load (box given by the tensor map) completing on `bar`.
__device__ __forceinline__ void load_4d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                        int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];" ::"r"(sa(dst)),
      "l"(map), "r"(sa(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// Warp-converged issue: the whole warp executes these with warp-uniform
// operands and one elected lane issues. The operands then stay in uniform
// registers; issuing from a lane-divergent branch (if (lane == 0)) makes the
// compiler wrap every TMA / MMA in an R2UR.BROADCAST waterfall loop (~60
// cycles per instruction).
__device__ __forceinline__ void mbar_expect_tx_e(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n}\n" ::"r"(sa(bar)),
      "r"(bytes)
      : "memory");
}

__device__ __forceinline__ void load_2d_e(const CUtensorMap* map, uint64_t* bar, void* dst, int x, int y) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];\n}\n" ::"r"(sa(dst)),
      "l"(map), "r"(sa(bar)), "r"(x), "r"(y)
      : "memory");
}

__device__ __forceinline__ void load_4d_e(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1, int c2,
                                          int c3) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2];\n}\n" ::"r"(sa(dst)),
      "l"(map), "r"(sa(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// ------------------------------------------------------------- clusters --

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}

// Address of `local` in the shared memory of cluster CTA `rank`.
__device__ __forceinline__ uint32_t map_rank(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(sa(local)), "r"(rank));
  return r;
}

__device__ __forceinline__ float ld_dsmem_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}

}  // namespace tma
}  // namespace psk

#include "../../include/psk.h"
namespace psk {
// TMA maps over a paged KV pool (decode_attn.cu), 128B-swizzled:
//  KV_BOX2D : 2D, [16 token x 64 dim] boxes (one half of a K or V tile);
//  KV_TILE3D: 3D (64 dim, 16 token, 2 halves), one box = a whole 4 KiB K or
//             V tile landing as [half0 | half1] x [16][128 B];
//  KV_PAGE4D: 4D (64 dim, 16 token, 2 halves, K|V), one box = the whole
//             8 KiB K+V of one (page, layer, head), landing as
//             [K half0 | K half1 | V half0 | V half1] x [16][128 B].
//  KV_PAGE4D_ALL: as KV_PAGE4D with all n_kv_heads heads' token rows in one
//             box (the page's whole K|V block of a layer, 64 KiB at 8 heads).
enum KvMapKind { KV_BOX2D = 0, KV_TILE3D = 1, KV_PAGE4D = 2, KV_PAGE4D_ALL = 3 };
int kv_tensor_map(const psk_kv_layout& kv, CUtensorMap* out, int kind = KV_BOX2D);
}  // namespace psk
