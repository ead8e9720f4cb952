// Error reporting, device queries and deterministic init kernels.
#include "common.cuh"

#include <stdarg.h>
#include <stdlib.h>

namespace psk {

static thread_local char g_last_error[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

// Counter-based Gaussian: two independent splitmix64 outputs keyed by
// (seed, index) feed a Box-Muller transform. Any element can be regenerated
// in isolation, so init is embarrassingly parallel and grid-size invariant.
__global__ void init_normal_bf16_kernel(__nv_bfloat16* __restrict__ dst, int64_t n,
                                        uint64_t seed, float stdv) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint64_t h1 = mix64(seed ^ mix64((uint64_t)i * 2ull + 0x632BE59BD9B4E019ull));
    uint64_t h2 = mix64(seed ^ mix64((uint64_t)i * 2ull + 1ull + 0x632BE59BD9B4E019ull));
    float u1 = (float)((h1 >> 40) + 1ull) * (1.0f / 16777216.0f);  // (0, 1]
    float u2 = (float)(h2 >> 40) * (1.0f / 16777216.0f);           // [0, 1)
    float z = sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
    dst[i] = f2bf(stdv * z);
  }
}

__global__ void fill_bf16_kernel(__nv_bfloat16* __restrict__ dst, int64_t n, float v) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  __nv_bfloat16 b = f2bf(v);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) dst[i] = b;
}

static unsigned long long* s_trace_buf = nullptr;
static int s_trace_cap = 0;

unsigned long long* trace_buffer(int n_ctas) {
  static const bool on = getenv("PSK_TRACE") != nullptr;
  if (!on) return nullptr;
  if (n_ctas > s_trace_cap) {
    if (s_trace_buf) cudaFree(s_trace_buf);
    cudaMalloc(&s_trace_buf, sizeof(unsigned long long) * 8 * n_ctas);
    s_trace_cap = n_ctas;
  }
  cudaMemset(s_trace_buf, 0, sizeof(unsigned long long) * 8 * n_ctas);
  return s_trace_buf;
}

void trace_report(const char* kernel, int n, int nph, const char* const* names) {
  cudaDeviceSynchronize();
  unsigned long long* h = (unsigned long long*)malloc(sizeof(unsigned long long) * 8 * n);
  cudaMemcpy(h, s_trace_buf, sizeof(unsigned long long) * 8 * n, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull;
  for (int i = 0; i < n; ++i)
    if (h[i * 8] && h[i * 8] < t0) t0 = h[i * 8];
  fprintf(stderr, "[trace %s] %d CTAs, us since first CTA entry: min / avg / max\n", kernel, n);
  for (int k = 0; k < nph; ++k) {
    double mn = 1e30, mx = 0, av = 0;
    int c = 0;
    for (int i = 0; i < n; ++i) {
      if (!h[i * 8 + k]) continue;
      double v = (double)(h[i * 8 + k] - t0) / 1000.0;
      mn = v < mn ? v : mn;
      mx = v > mx ? v : mx;
      av += v;
      ++c;
    }
    if (c) fprintf(stderr, "  %-14s %8.2f %8.2f %8.2f  (%d CTAs)\n", names[k], mn, av / c, mx, c);
  }
  free(h);
}

static int g_sm_budget = 0;

int device_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return sms;
}

int sm_budget() {
  const int d = device_sms();
  return g_sm_budget > 0 && g_sm_budget < d ? g_sm_budget : d;
}

static int grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  if (g > 148 * 16) g = 148 * 16;
  if (g < 1) g = 1;
  return (int)g;
}

}  // namespace psk

extern "C" {

int psk_abi_version(void) { return PSK_ABI_VERSION; }

const char* psk_last_error(void) { return psk::g_last_error; }

int psk_sm_count(int device, int32_t* out) {
  PSK_CHECK_ARG(out != nullptr, "psk_sm_count: null out");
  int v = 0;
  PSK_CUDA_TRY(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
  *out = v;
  return PSK_OK;
}

int psk_set_sm_budget(int32_t n) {
  PSK_CHECK_ARG(n >= 0, "psk_set_sm_budget: negative budget");
  PSK_CHECK_ARG(n == 0 || n >= 2, "psk_set_sm_budget: budget must be 0 (all SMs) or >= 2");
  psk::g_sm_budget = n;
  return PSK_OK;
}

int psk_get_sm_budget(int32_t* out) {
  PSK_CHECK_ARG(out != nullptr, "psk_get_sm_budget: null out");
  *out = psk::sm_budget();
  return PSK_OK;
}

int psk_init_normal_bf16(void* dst, int64_t n, uint64_t seed, float stdv, void* stream) {
  PSK_CHECK_ARG(dst != nullptr && n >= 0, "psk_init_normal_bf16: bad args");
  if (n == 0) return PSK_OK;
  psk::init_normal_bf16_kernel<<<psk::grid_for(n, 256), 256, 0, psk::as_stream(stream)>>>(
      reinterpret_cast<__nv_bfloat16*>(dst), n, seed, stdv);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

int psk_fill_bf16(void* dst, int64_t n, float value, void* stream) {
  PSK_CHECK_ARG(dst != nullptr && n >= 0, "psk_fill_bf16: bad args");
  if (n == 0) return PSK_OK;
  psk::fill_bf16_kernel<<<psk::grid_for(n, 256), 256, 0, psk::as_stream(stream)>>>(
      reinterpret_cast<__nv_bfloat16*>(dst), n, value);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}

}  // extern "C"
