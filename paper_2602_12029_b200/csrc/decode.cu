// Decode-module step kernels: embedding, RMSNorm, RoPE + paged KV append
// and greedy argmax (the grouped GEMV K5 is in gemv.cu, the shared-prefix
// decode attention K6 in decode_attn.cu).
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
#include <stdlib.h>

namespace psk {
namespace dec {

constexpr int HD = 128;
constexpr int PT = 16;  // tokens per KV page (= kvstore block_size)

// ------------------------------------------------------------- embedding --

__global__ void embed_rows_kernel(psk_decode_batch b, const __nv_bfloat16* const* embed, int d,
                                  float* __restrict__ h) {
  pdl_wait();  // first kernel of a step: the previous step is fully done
  pdl_trigger();
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

// One CTA (256 threads) per row; the row stays in registers between the
// sum of squares and the scaled store (one HBM read of h), gamma is read
// before the PDL wait (weights never depend on the previous kernel).
constexpr int NORM_THREADS = 256;
constexpr int NORM_VPT = 8;  // float4 per thread: d <= 8192

__global__ void __launch_bounds__(NORM_THREADS) rmsnorm_rows_kernel(const float* __restrict__ h, int d,
                                    const __nv_bfloat16* const* gamma, const int32_t* row_mod,
                                    float eps, __nv_bfloat16* __restrict__ out) {
  __shared__ float s_red[32];
  pdl_trigger();
  const int r = blockIdx.x;
  const __nv_bfloat16* g = gamma[row_mod ? row_mod[r] : 0];
  const int n4 = d >> 2;
  uint2 gv[NORM_VPT];
#pragma unroll
  for (int u = 0; u < NORM_VPT; ++u) {
    const int i = threadIdx.x + u * NORM_THREADS;
    gv[u] = i < n4 ? __ldg(reinterpret_cast<const uint2*>(g) + i) : make_uint2(0, 0);
  }
  pdl_wait();
  const float4* x = reinterpret_cast<const float4*>(h + (int64_t)r * d);
  float4 v[NORM_VPT];
  float ss = 0.f;
#pragma unroll
  for (int u = 0; u < NORM_VPT; ++u) {
    const int i = threadIdx.x + u * NORM_THREADS;
    v[u] = i < n4 ? x[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int u = 0; u < NORM_VPT; ++u) ss += v[u].x * v[u].x + v[u].y * v[u].y + v[u].z * v[u].z + v[u].w * v[u].w;
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < (NORM_THREADS >> 5) ? s_red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) s_red[0] = t;
  }
  __syncthreads();
  const float inv = rsqrtf(s_red[0] / (float)d + eps);
  uint2* o = reinterpret_cast<uint2*>(out + (int64_t)r * d);
#pragma unroll
  for (int u = 0; u < NORM_VPT; ++u) {
    const int i = threadIdx.x + u * NORM_THREADS;
    if (i >= n4) continue;
    const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gv[u].x));
    const float2 c = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&gv[u].y));
    const __nv_bfloat162 o01 = __floats2bfloat162_rn(v[u].x * inv * a.x, v[u].y * inv * a.y);
    const __nv_bfloat162 o23 = __floats2bfloat162_rn(v[u].z * inv * c.x, v[u].w * inv * c.y);
    uint2 w;
    w.x = *reinterpret_cast<const uint32_t*>(&o01);
    w.y = *reinterpret_cast<const uint32_t*>(&o23);
    o[i] = w;
  }
}

// ---------------------------------------------------- RoPE + KV append ---


// One CTA per row, 64 x 8 threads: thread (i, j) rotates dims (i, i + 64) of
// heads j, j + 8, ... (q heads, then k), copies v; all of a thread's loads
// are independent (no per-head dependent chain).
constexpr int ROPE_HG = 8;

__global__ void __launch_bounds__(64 * ROPE_HG) rope_append_kernel(psk_decode_batch b, const float* __restrict__ qkv,
                                                                  int nq, const float* __restrict__ rope, int layer,
                                                                  psk_kv_layout kv, __nv_bfloat16* __restrict__ q_rot) {
  // the attention kernel (PDL-launched next) may start its table prologue now
  asm volatile("griddepcontrol.launch_dependents;");
  const int r = blockIdx.x;
  const int nkv = kv.n_kv_heads;
  const int idx = b.priv_len[r];
  const int pos = b.sess_len[b.row_sess[r]] + idx;
  const int page = b.row_pages[(int64_t)r * b.max_row_pages + idx / PT];
  const int off = idx % PT;
  const float* row = qkv + (int64_t)r * (nq + 2 * nkv) * HD;
  const float* cs = rope + (int64_t)pos * HD;  // [64][2]
  const int i = threadIdx.x & 63, j = threadIdx.x >> 6;
  const float c = cs[2 * i], s = cs[2 * i + 1];
  pdl_wait();  // qkv comes from the GEMV just before
  // q and k heads: rotate-half
#pragma unroll 4
  for (int h = j; h < nq + nkv; h += ROPE_HG) {
    float y1, y2;
    rope_pair(row[h * HD + i], row[h * HD + i + 64], c, s, y1, y2);
    __nv_bfloat16* d = h < nq ? q_rot + ((int64_t)r * nq + h) * HD : kv_row(kv, page, layer, 0, h - nq, off);
    d[i] = f2bf(y1);
    d[i + 64] = f2bf(y2);
  }
  for (int h = j; h < nkv; h += ROPE_HG) {
    const float* vr = row + (nq + nkv + h) * HD;
    __nv_bfloat16* vd = kv_row(kv, page, layer, 1, h, off);
    vd[i] = f2bf(vr[i]);
    vd[i + 64] = f2bf(vr[i + 64]);
  }
}

// ---------------------------------------------------------------- argmax --

// Block-wide first-maximum argmax of x[0, V) (tf.argMax / torch.argmax tie
// rule); the result is valid in thread 0.
__device__ int block_argmax(const float* __restrict__ x, int V, float* s_v, int* s_i) {
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  // ties resolve to the lowest index (first maximum, as the reference argmax)
#define PSK_TAKE(v, i) \
  if ((v) > bv || ((v) == bv && (i) < bi)) { bv = (v); bi = (i); }
  int tail = 0;
  if ((V & 3) == 0) {
    // 4 independent float4 loads in flight per thread (the logits sit in L2)
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const int V4 = V >> 2, step = blockDim.x;
    int i = threadIdx.x;
    for (; i + 3 * step < V4; i += 4 * step) {
      float4 q[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) q[u] = __ldg(x4 + i + u * step);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = (i + u * step) * 4;
        PSK_TAKE(q[u].x, e) PSK_TAKE(q[u].y, e + 1) PSK_TAKE(q[u].z, e + 2) PSK_TAKE(q[u].w, e + 3)
      }
    }
    for (; i < V4; i += step) {
      const float4 q = __ldg(x4 + i);
      PSK_TAKE(q.x, 4 * i) PSK_TAKE(q.y, 4 * i + 1) PSK_TAKE(q.z, 4 * i + 2) PSK_TAKE(q.w, 4 * i + 3)
    }
    tail = V;
  }
  for (int i = tail + threadIdx.x; i < V; i += blockDim.x) PSK_TAKE(__ldg(x + i), i)
#undef PSK_TAKE
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
  }
  return bi;
}

__global__ void argmax_advance_kernel(psk_decode_batch b, const float* __restrict__ logits, int V,
                                      int32_t* __restrict__ out_tokens, int max_new) {
  __shared__ float s_v[32];
  __shared__ int s_i[32];
  pdl_wait();
  const int r = blockIdx.x;
  const int bi = block_argmax(logits + (int64_t)r * V, V, s_v, s_i);
  if (threadIdx.x == 0) {
    const int k = b.priv_len[r];
    if (out_tokens && k < max_new) out_tokens[(int64_t)r * max_new + k] = bi;
    b.tokens[r] = bi;
    // saturate at the row's page capacity: idle continuous-batching slots keep
    // stepping without ever indexing past their private page table
    b.priv_len[r] = min(k + 1, b.max_row_pages * PT - 1);
  }
}

__global__ void argmax_rows_kernel(const float* __restrict__ logits, int V, int32_t* __restrict__ out) {
  __shared__ float s_v[32];
  __shared__ int s_i[32];
  const int bi = block_argmax(logits + (int64_t)blockIdx.x * V, V, s_v, s_i);
  if (threadIdx.x == 0) out[blockIdx.x] = bi;
}

}  // namespace dec
}  // namespace psk

using namespace psk::dec;


extern "C" {

int psk_embed_rows(const psk_decode_batch* b, const void* const* embed, int32_t d, float* h,
                   void* stream) {
  PSK_CHECK_ARG(b && embed && h && d % 8 == 0, "psk_embed_rows: bad args");
  if (b->n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(embed_rows_kernel, dim3(b->n_rows), dim3(128), 0, psk::as_stream(stream),
                               *b, reinterpret_cast<const __nv_bfloat16* const*>(embed), d, h));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_rmsnorm_rows(const float* h, int32_t n_rows, int32_t d, const void* const* gamma,
                     const int32_t* row_mod, float eps, void* out, void* stream) {
  PSK_CHECK_ARG(h && gamma && out && d % 4 == 0 && n_rows >= 0 && d <= 4 * NORM_THREADS * NORM_VPT,
                "psk_rmsnorm_rows: bad args (d %% 4 == 0, d <= %d)", 4 * NORM_THREADS * NORM_VPT);
  if (n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(rmsnorm_rows_kernel, dim3(n_rows), dim3(NORM_THREADS), 0, psk::as_stream(stream),
                               h, d, reinterpret_cast<const __nv_bfloat16* const*>(gamma), row_mod,
                               eps, reinterpret_cast<__nv_bfloat16*>(out)));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_rope_append(const psk_decode_batch* b, const float* qkv, int32_t n_q_heads,
                    const float* rope, int32_t layer, psk_kv_layout kv, void* q_rot, void* stream) {
  PSK_CHECK_ARG(b && qkv && rope && q_rot && kv.head_dim == HD && kv.page_tokens == PT,
                "psk_rope_append: bad args (head_dim must be 128, page_tokens 16)");
  if (b->n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(rope_append_kernel, dim3(b->n_rows), dim3(64 * ROPE_HG), 0, psk::as_stream(stream),
                               *b, qkv, n_q_heads, rope, layer, kv,
                               reinterpret_cast<__nv_bfloat16*>(q_rot)));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_argmax_advance(const psk_decode_batch* b, const float* logits, int32_t vocab,
                       int32_t* out_tokens, int32_t max_new, void* stream) {
  PSK_CHECK_ARG(b && logits && vocab > 0, "psk_argmax_advance: bad args");
  if (b->n_rows == 0) return PSK_OK;
  PSK_CUDA_TRY(psk::launch_pdl(argmax_advance_kernel, dim3(b->n_rows), dim3(1024), 0,
                               psk::as_stream(stream), *b, logits, vocab, out_tokens, max_new));
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_argmax_rows(const float* logits, int32_t n_rows, int32_t vocab, int32_t* out, void* stream) {
  PSK_CHECK_ARG(logits && out && vocab > 0 && n_rows >= 0, "psk_argmax_rows: bad args");
  if (n_rows == 0) return PSK_OK;
  psk::dec::argmax_rows_kernel<<<n_rows, 1024, 0, psk::as_stream(stream)>>>(logits, vocab, out);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // extern "C"
