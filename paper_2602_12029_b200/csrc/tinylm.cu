// TinyLM forward on the GPU over a paged prompt cache (psk_tiny_forward).
//
// The reference's own model (frontend/src/model.ts:112-331): token +
// previous-token + learned position embeddings, L x [LayerNorm -> Q/K/V ->
// causal softmax attention over [cached prefix | new tokens] -> Wo ->
// residual -> LayerNorm -> GELU-tanh MLP (biases) -> residual], final
// LayerNorm -> head. fp32 like the reference (tfjs is fp32).
//
// B200 form: one launch per forward; a sequence is one 8-CTA thread-block
// cluster that runs every layer, each phase (embeddings, LayerNorm rows,
// GEMM output tiles, attention (head, token-phase) units) split over the
// cluster's CTAs with a cluster barrier between phases (a 64-256 wide
// model is latency-bound; activations stay in L2-resident scratch). The prompt cache is
// paged instead of model.ts's concatenated [B, H, S, hd] tensors: 16-token
// pages [page][layer][K|V][head][16][hd], a block table per sequence, so a
// decode module's forward reads the frozen base's pages of the shared
// prefix in place (PromptCache.slice, model.ts:58-70, becomes a shorter
// block table) and appends its own tokens to its own pages.
#include "common.cuh"
#include "psk.h"

namespace psk {
namespace tiny {

constexpr int PT = 16;
constexpr int THREADS = 256;
constexpr int WARPS = THREADS / 32;
constexpr int NPTR = 12;  // per-layer parameter pointers (psk.h)
constexpr int CL = 8;     // CTAs per sequence (one thread-block cluster)

// Phase boundary of a sequence's forward: every CTA of the cluster has
// finished the phase and its global writes are visible (release / acquire
// at cluster scope).
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct Args {
  psk_tiny_model m;
  int T, S0, max_pages;
  int staged;  // attention K / V rows staged in shared memory (else read from the pages)
  const int32_t* tokens;
  const int32_t* prev_first;
  const int32_t* table;
  float* kv;
  float* scratch;
  float* logits;
};

// LayerNorm of T rows of width d, eps 1e-5, biased variance (model.ts:120-123): warp per row.
__device__ void layer_norm(const float* in, float* out, const float* g, const float* b, int T, int d, int rank) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = rank * WARPS + warp; t < T; t += CL * WARPS) {
    const float* x = in + (int64_t)t * d;
    float s = 0.f;
    for (int c = lane; c < d; c += 32) s += x[c];
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / d;
    float v = 0.f;
    for (int c = lane; c < d; c += 32) {
      const float e = x[c] - mean;
      v += e * e;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const float inv = 1.f / sqrtf(v / d + 1e-5f);
    for (int c = lane; c < d; c += 32) out[(int64_t)t * d + c] = (x[c] - mean) * inv * g[c] + b[c];
  }
}

__device__ __forceinline__ float gelu_tanh(float x) {  // model.ts:114-118
  return 0.5f * x * (1.f + tanhf((x + 0.044715f * x * x * x) * 0.7978845608028654f));
}

// Y[t, n] (op)= sum_k X[t, k] W[k, n] (+ bias[n]) for t < T, n < N: 64 x 64
// output tiles through shared memory (16-deep k slabs of X and W, the next
// slab's loads in flight under this one's FMAs), each thread a 4 x 4
// register block; k accumulates in order. Call with every thread of the CTA.
constexpr int BM = 64, BN = 64, BK = 16;
struct Tiles {
  float A[BK][BM + 4], B[BK][BN];
};
template <class Out>
__device__ void matmul(Tiles& tl, int rank, const float* X, int T, int K, const float* W, int N, const float* bias,
                       Out out) {
  auto& As = tl.A;
  auto& Bs = tl.B;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int tn = (N + BN - 1) / BN, tiles = ((T + BM - 1) / BM) * tn;
  for (int ti = rank; ti < tiles; ti += CL) {  // output tiles split over the cluster
    const int m0 = (ti / tn) * BM, n0 = (ti % tn) * BN;
    {
      float acc[4][4] = {};
      // the next k slab is loaded into registers while this one computes
      constexpr int LA = BM * BK / THREADS, LB = BK * BN / THREADS;
      float ra[LA], rb[LB];
      auto load = [&](int k0) {
#pragma unroll
        for (int u = 0; u < LA; ++u) {
          const int i = threadIdx.x + u * THREADS, r = i / BK, c = i - r * BK, t = m0 + r, k = k0 + c;
          ra[u] = (t < T && k < K) ? X[(int64_t)t * K + k] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int i = threadIdx.x + u * THREADS, r = i / BN, c = i - r * BN, k = k0 + r, n = n0 + c;
          rb[u] = (k < K && n < N) ? W[(int64_t)k * N + n] : 0.f;
        }
      };
      load(0);
      for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int u = 0; u < LA; ++u) {
          const int i = threadIdx.x + u * THREADS, r = i / BK;
          As[i - r * BK][r] = ra[u];
        }
#pragma unroll
        for (int u = 0; u < LB; ++u) {
          const int i = threadIdx.x + u * THREADS, r = i / BN;
          Bs[r][i - r * BN] = rb[u];
        }
        __syncthreads();
        if (k0 + BK < K) load(k0 + BK);
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
          float a4[4], b4[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            a4[i] = As[kk][ty * 4 + i];
            b4[i] = Bs[kk][tx * 4 + i];
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a4[i], b4[j], acc[i][j]);
        }
        __syncthreads();
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int t = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
          if (t < T && n < N) out(t, n, acc[i][j] + (bias ? bias[n] : 0.f));
        }
    }
  }
}

__global__ void __launch_bounds__(THREADS, 1) tiny_forward_kernel(const Args a) {
  extern __shared__ float s_p[];  // one head's K / V rows, then per warp: probabilities + q
  __shared__ Tiles tiles;
  const psk_tiny_model& m = a.m;
  const int b = blockIdx.x / CL, rank = blockIdx.x % CL, T = a.T, S0 = a.S0, d = m.width, H = m.heads, hd = d / H;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t page_f = (int64_t)m.layers * 2 * PT * d;  // floats per page
  float* x = a.scratch + (int64_t)b * 8 * T * d;
  float* xn = x + (int64_t)T * d;
  float* q = xn + (int64_t)T * d;
  float* ctx = q + (int64_t)T * d;
  float* hid = ctx + (int64_t)T * d;  // [T][4d]
  const int32_t* tok = a.tokens + (int64_t)b * T;
  const int32_t* tab = a.table + (int64_t)b * a.max_pages;
  // embeddings (model.ts:262-276): previous token of position 0 = the last
  // token the cache covers (-1: none -> no prev-token term)
  for (int i = rank * THREADS + threadIdx.x; i < T * d; i += CL * THREADS) {
    const int t = i / d, c = i - t * d;
    const int prev = t > 0 ? tok[t - 1] : a.prev_first[b];
    float v = m.tok_emb[(int64_t)tok[t] * d + c] + (prev >= 0 ? m.prev_emb[(int64_t)prev * d + c] : 0.f);
    x[i] = v + m.pos_emb[(int64_t)(S0 + t) * d + c];
  }
  cluster_sync();
  const float scale = 1.f / sqrtf((float)hd);
  for (int l = 0; l < m.layers; ++l) {
    const float* const* w = m.blocks + (int64_t)l * NPTR;
    layer_norm(x, xn, w[0], w[1], T, d, rank);
    cluster_sync();
    matmul(tiles, rank, xn, T, d, w[2], d, nullptr, [&](int t, int n, float v) { q[(int64_t)t * d + n] = v; });
    // K / V of the new tokens -> their pages (positions S0 .. S0 + T - 1)
    for (int kv = 0; kv < 2; ++kv)
      matmul(tiles, rank, xn, T, d, w[3 + kv], d, nullptr, [&](int t, int n, float v) {
        const int pos = S0 + t, hh = n / hd;
        float* pg = a.kv + (int64_t)tab[pos / PT] * page_f;
        pg[(((int64_t)(l * 2 + kv) * H + hh) * PT + pos % PT) * hd + (n - hh * hd)] = v;
      });
    cluster_sync();
    // attention, head by head: the head's K / V rows for keys 0 .. S0+T-1
    // staged in shared memory ([key][hd + 1]: conflict-free for a lane per
    // key and for a lane per dim), then a warp per new token t over keys
    // 0 .. S0 + t (the reference's -1e9 mask on later keys is an exact zero
    // after exp)
    // (a head too large for shared memory is read from its pages instead)
    const int S_all = S0 + T, hs = hd + 1;
    float* Ks = s_p;
    float* Vs = Ks + (a.staged ? (int64_t)S_all * hs : 0);
    float* pr = Vs + (a.staged ? (int64_t)S_all * hs : 0) + (int64_t)warp * (m.context + hd);
    float* qs = pr + m.context;
    // units (head, token phase) over the cluster: a head's tokens are split
    // ts::hsplit among hsplit CTAs when the cluster has more CTAs than heads
    const int hsplit = CL % H == 0 ? CL / H : 1;
    for (int u = rank; u < H * hsplit; u += CL) {
      const int hh = u / hsplit, ts = u % hsplit;
      auto kv_row = [&](int j, int kv) -> const float* {
        return a.kv + (int64_t)tab[j / PT] * page_f + (((int64_t)(l * 2 + kv) * H + hh) * PT + j % PT) * hd;
      };
      for (int i = threadIdx.x; a.staged && i < S_all * hd; i += THREADS) {
        const int j = i / hd, e = i - j * hd;
        const float* pg = a.kv + (int64_t)tab[j / PT] * page_f + (((int64_t)(l * 2) * H + hh) * PT + j % PT) * hd + e;
        Ks[j * hs + e] = pg[0];
        Vs[j * hs + e] = pg[(int64_t)H * PT * hd];  // V sits H tiles after K
      }
      __syncthreads();
      for (int t = ts + warp * hsplit; t < T; t += WARPS * hsplit) {
        const int S = S0 + t + 1;
        for (int e = lane; e < hd; e += 32) qs[e] = q[(int64_t)t * d + hh * hd + e];
        __syncwarp();
        float mx = -INFINITY;
        for (int j = lane; j < S; j += 32) {
          const float* kr = a.staged ? Ks + j * hs : kv_row(j, 0);
          float sc = 0.f;
          for (int e = 0; e < hd; ++e) sc = fmaf(qs[e], kr[e], sc);
          sc *= scale;
          pr[j] = sc;
          mx = fmaxf(mx, sc);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float sum = 0.f;
        for (int j = lane; j < S; j += 32) {
          const float ex = expf(pr[j] - mx);
          pr[j] = ex;
          sum += ex;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
        __syncwarp();
        const float inv = 1.f / sum;
        for (int e = lane; e < hd; e += 32) {
          float acc = 0.f;
          if (a.staged)
            for (int j = 0; j < S; ++j) acc = fmaf(pr[j], Vs[j * hs + e], acc);
          else
            for (int j = 0; j < S; ++j) acc = fmaf(pr[j], kv_row(j, 1)[e], acc);
          ctx[(int64_t)t * d + hh * hd + e] = acc * inv;
        }
        __syncwarp();
      }
      __syncthreads();
    }
    cluster_sync();
    matmul(tiles, rank, ctx, T, d, w[5], d, nullptr, [&](int t, int n, float v) { x[(int64_t)t * d + n] += v; });
    cluster_sync();
    layer_norm(x, xn, w[6], w[7], T, d, rank);
    cluster_sync();
    matmul(tiles, rank, xn, T, d, w[8], 4 * d, w[9], [&](int t, int n, float v) { hid[(int64_t)t * 4 * d + n] = gelu_tanh(v); });
    cluster_sync();
    matmul(tiles, rank, hid, T, 4 * d, w[10], d, w[11], [&](int t, int n, float v) { x[(int64_t)t * d + n] += v; });
    cluster_sync();
  }
  layer_norm(x, xn, m.lnf_g, m.lnf_b, T, d, rank);
  cluster_sync();
  float* lg = a.logits + (int64_t)b * T * m.vocab;
  matmul(tiles, rank, xn, T, d, m.head, m.vocab, nullptr, [&](int t, int n, float v) { lg[(int64_t)t * m.vocab + n] = v; });
}

}  // namespace tiny
}  // namespace psk

extern "C" {

int psk_tiny_scratch_floats(const psk_tiny_model* m, int32_t batch, int32_t n_new, int64_t* out) {
  PSK_CHECK_ARG(m && out && batch >= 0 && n_new >= 0, "psk_tiny_scratch_floats: bad args");
  *out = (int64_t)batch * 8 * n_new * m->width;
  return PSK_OK;
}

int psk_tiny_forward(const psk_tiny_model* m, int32_t batch, int32_t n_new, int32_t past_len,
                     const int32_t* tokens, const int32_t* prev_first, const int32_t* block_table,
                     int32_t max_pages, float* kv_pages, int64_t n_pages, float* scratch, float* logits,
                     void* stream) {
  using namespace psk::tiny;
  PSK_CHECK_ARG(m && tokens && prev_first && block_table && kv_pages && scratch && logits && m->blocks,
                "psk_tiny_forward: null argument");
  PSK_CHECK_ARG(m->layers > 0 && m->width > 0 && m->heads > 0 && m->width % m->heads == 0 && m->vocab > 0,
                "width %d not divisible by heads %d", m->width, m->heads);
  PSK_CHECK_ARG(batch > 0 && n_new > 0 && past_len >= 0, "psk_tiny_forward: empty batch");
  PSK_CHECK_ARG(past_len + n_new <= m->context, "sequence length %d exceeds context %d", past_len + n_new,
                m->context);
  PSK_CHECK_ARG((int64_t)max_pages * PT >= past_len + n_new && n_pages > 0,
                "block table of %d pages cannot hold %d tokens", max_pages, past_len + n_new);
  const int hd = m->width / m->heads;
  const size_t rows = sizeof(float) * WARPS * (size_t)(m->context + hd);
  const size_t kv_stage = sizeof(float) * 2 * (size_t)(past_len + n_new) * (hd + 1);
  const bool staged = rows + kv_stage <= 200 * 1024;
  const size_t smem = staged ? rows + kv_stage : rows;
  PSK_CHECK_ARG(smem <= 200 * 1024, "context %d x head dim %d too large for the attention row buffers", m->context,
                hd);
  static size_t smem_set = 0;
  if (smem > 48 * 1024 && smem > smem_set) {
    PSK_CUDA_TRY(cudaFuncSetAttribute(tiny_forward_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    smem_set = smem;
  }
  Args a;
  a.m = *m;
  a.T = n_new;
  a.staged = staged;
  a.S0 = past_len;
  a.max_pages = max_pages;
  a.tokens = tokens;
  a.prev_first = prev_first;
  a.table = block_table;
  a.kv = kv_pages;
  a.scratch = scratch;
  a.logits = logits;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)batch * CL);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = psk::as_stream(stream);
  cfg.attrs = at;
  cfg.numAttrs = 1;
  PSK_CUDA_TRY(cudaLaunchKernelEx(&cfg, tiny_forward_kernel, a));
  return PSK_OK;
}

}  // extern "C"
