// K8 — KV page copy (prefill -> decode handoff building block).
//
// Replaces the modelled transfer of src/prefillsim/costs.py:66-83 (bytes /
// bandwidth x staging penalty) that cluster.py:376-412 schedules per
// request. Cross-process handoffs go through NCCL P2P of whole pages
// (transfer.py); this kernel moves pages between two page pools addressable
// from the launching device — the same pool (tail-page copies), another pool
// on the same GPU, or a peer GPU's pool mapped with peer access (SM-driven
// NVLink stores). One CTA streams whole pages with 16-byte vector loads and
// stores, several pages in flight per SM; the copy is HBM/NVLink bound.
#include "common.cuh"

namespace psk {
namespace xfer {

__global__ void __launch_bounds__(512) copy_pages_kernel(const uint4* __restrict__ src_base,
                                                         uint4* __restrict__ dst_base,
                                                         const int32_t* __restrict__ src_pages,
                                                         const int32_t* __restrict__ dst_pages,
                                                         int n, int64_t page_vec) {
  for (int i = blockIdx.y; i < n; i += gridDim.y) {
    const uint4* s = src_base + (int64_t)src_pages[i] * page_vec;
    uint4* d = dst_base + (int64_t)dst_pages[i] * page_vec;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; e + 3 * stride < page_vec; e += 4 * stride) {
      const uint4 a = ld_stream_v4(s + e), b = ld_stream_v4(s + e + stride);
      const uint4 c = ld_stream_v4(s + e + 2 * stride), f = ld_stream_v4(s + e + 3 * stride);
      d[e] = a;
      d[e + stride] = b;
      d[e + 2 * stride] = c;
      d[e + 3 * stride] = f;
    }
    for (; e < page_vec; e += stride) d[e] = ld_stream_v4(s + e);
  }
}

}  // namespace xfer
}  // namespace psk

extern "C" int psk_kv_copy_pages(const void* src_base, void* dst_base, const int32_t* src_pages,
                                 const int32_t* dst_pages, int32_t n_pages, int64_t page_bytes,
                                 void* stream) {
  PSK_CHECK_ARG(src_base && dst_base && src_pages && dst_pages && n_pages >= 0 && page_bytes % 16 == 0,
                "psk_kv_copy_pages: bad args");
  if (n_pages == 0) return PSK_OK;
  const int64_t vec = page_bytes / 16;
  int xb = (int)((vec + 512 * 4 - 1) / (512 * 4));
  if (xb > 8) xb = 8;
  int yb = n_pages < 296 ? n_pages : 296;
  psk::xfer::copy_pages_kernel<<<dim3(xb, yb), 512, 0, psk::as_stream(stream)>>>(
      reinterpret_cast<const uint4*>(src_base), reinterpret_cast<uint4*>(dst_base), src_pages, dst_pages,
      n_pages, vec);
  PSK_LAUNCH_CHECK();
  return PSK_OK;
}
