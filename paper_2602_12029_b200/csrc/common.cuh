// Shared helpers for the PrefillShare B200 kernels (sm_100a only).
//
// Every extern "C" entry point returns 0 on success or a negative PSK_E*
// code; the message for the last failure on the calling thread is kept for
// psk_last_error(). No entry point allocates device memory on a hot call:
// all buffers are caller-owned (torch tensors on the Python side).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <stdio.h>

#include "../../include/psk.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_2602_12029_b200 kernels target sm_100a only"
#endif

namespace psk {

void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// SMs the persistent kernels size their grids for: the device's count, or
// the budget set with psk_set_sm_budget (a spatial share of the GPU for
// kernels that run beside another stream's work, e.g. prefill beside decode).
int sm_budget();
int device_sms();

}  // namespace psk

#define PSK_CHECK_ARG(cond, ...)                       \
  do {                                                 \
    if (!(cond)) {                                     \
      psk::set_error(__VA_ARGS__);                     \
      return PSK_EINVAL;                               \
    }                                                  \
  } while (0)

#define PSK_CUDA_TRY(expr)                                                    \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      psk::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr,              \
                     cudaGetErrorString(_e));                                 \
      return PSK_ECUDA;                                                       \
    }                                                                         \
  } while (0)

#define PSK_LAUNCH_CHECK() PSK_CUDA_TRY(cudaGetLastError())

namespace psk {

// Programmatic dependent launch (PDL). Kernels of a decode step trigger their
// dependents early and wait on the predecessor grid only before reading data
// produced within the step; data that is constant during a step (weights,
// page tables, lengths) may be read before the wait. The first kernel of a
// step waits before triggering, so nothing of step t+1 overlaps step t.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t stream, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ float bf2f(__nv_bfloat16 x) { return __bfloat162float(x); }
__device__ __forceinline__ __nv_bfloat16 f2bf(float x) { return __float2bfloat16_rn(x); }

// Unpack 8 bf16 held in a 16-byte vector into fp32.
__device__ __forceinline__ void bf16x8_to_f32(const uint4& v, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}

// Rotate-half RoPE (Llama) of the pair (x1, x2) = dims (i, i + 64) of a
// head: y1 = x1 c - x2 s, y2 = x2 c + x1 s. Explicit roundings, so every
// decode kernel that appends K (psk_rope_append, the fused K5-TC QKV
// epilogue) produces the same bits.
__device__ __forceinline__ void rope_pair(float x1, float x2, float c, float s, float& y1, float& y2) {
  y1 = __fmaf_rn(x1, c, -__fmul_rn(x2, s));
  y2 = __fmaf_rn(x2, c, __fmul_rn(x1, s));
}

// bf16 K (kvsel 0) or V (1) row of (page, layer, kv head, token) in the
// paged cache: page[layer][K|V][kv_head][token][head_dim].
__device__ __forceinline__ __nv_bfloat16* kv_row(const psk_kv_layout& kv, int32_t page, int layer, int kvsel,
                                                 int head, int tok) {
  return reinterpret_cast<__nv_bfloat16*>(kv.base) + (int64_t)page * kv.page_elems +
         ((((int64_t)layer * 2 + kvsel) * kv.n_kv_heads + head) * kv.page_tokens + tok) * kv.head_dim;
}

__device__ __forceinline__ uint4 f32_to_bf16x8(const float* f) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

// Streaming 128-bit load that does not allocate in L1 (weights / KV pages are
// read once per step).
__device__ __forceinline__ uint4 ld_stream_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// Phase tracing (debug/tuning; off unless PSK_TRACE is set in the
// environment): thread 0 of each CTA stamps %globaltimer at up to 8 phases.
static __device__ unsigned long long* g_trace = nullptr;  // one per translation unit
__device__ __forceinline__ void trace_stamp(int k) {
  unsigned long long* t = g_trace;
  if (t != nullptr && threadIdx.x == 0) {
    unsigned long long v;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
    t[(blockIdx.x + (size_t)blockIdx.y * gridDim.x) * 8 + k] = v;
  }
}
// Host: trace_buffer() returns a zeroed device buffer for n CTAs (nullptr
// when PSK_TRACE is unset); trace_report() prints per-phase min/avg/max (us
// since the first CTA's stamp 0) and disarms.
unsigned long long* trace_buffer(int n_ctas);
void trace_report(const char* kernel, int n_ctas, int n_phases, const char* const* names);
static inline bool trace_arm(int n_ctas) {
  unsigned long long* b = trace_buffer(n_ctas);
  if (!b) return false;
  cudaMemcpyToSymbol(g_trace, &b, sizeof(void*));
  return true;
}
static inline void trace_disarm() {
  unsigned long long* nul = nullptr;
  cudaMemcpyToSymbol(g_trace, &nul, sizeof(void*));
}

// 2^x on the MUFU (ex2.approx.ftz): 2^-inf = 0, no denormal range fix-up
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA pipe (the MUFU ex2 unit is the softmax limiter in K3):
// x = n + f with n = rint(x) via the 1.5 * 2^23 magic add, 2^f on
// [-0.5, 0.5] by a degree-3 minimax polynomial (max rel err 7.5e-5, far
// below bf16 P's 2^-8), n added into the exponent bits. Inputs are clamped
// at -125 (masked -inf scores give ~2^-125, negligible in sums of >= 1).
__device__ __forceinline__ float exp2_fma(float x) {
  x = fmaxf(x, -125.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05517167f, f, 0.24261115f), f, 0.69326097f), f, 0.99992806f);
  return __int_as_float(__float_as_int(p) + ((__float_as_int(t) - 0x4B400000) << 23));
}

// bar.sync on a named barrier (id 1..15) among `threads` threads (multiple of 32)
__device__ __forceinline__ void named_barrier_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__host__ __device__ __forceinline__ uint64_t splitmix64_next(uint64_t& state) {
  state += 0x9E3779B97F4A7C15ull;
  uint64_t z = state;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

}  // namespace psk
