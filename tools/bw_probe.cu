// HBM read-stream probe: what a weight-streaming kernel can get out of this
// B200 with different access patterns (build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a -o bw_probe tools/bw_probe.cu).
//   bulk  — one producer lane per CTA issues cp.async.bulk into a ring of
//           `stages` x `stage_kb` KiB; stage = `rows` pieces of (stage/rows)
//           bytes taken from rows `row_kb` KiB apart (rows=1: contiguous)
//   ldg   — every thread streams 16 B loads, `unroll` in flight
//   tma   — the K5-TC weight pattern: a bf16 [rows][4096] matrix streamed as
//           SW128 2-D boxes of 128 rows x 64 columns (128 B per row), `nbox`
//           consecutive k-chunk boxes per stage
#include <cuda.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void bulk_kernel(const char* __restrict__ src, int64_t bytes, int stages, int stage_bytes,
                            int rows, int64_t row_stride, float* sink) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(nw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  // unit = one stage worth of data: `rows` pieces of piece bytes, row_stride apart
  const int piece = stage_bytes / rows;
  const int64_t group_bytes = row_stride * rows;  // a group of `rows` rows
  const int64_t units_per_group = row_stride / piece;
  const int64_t units = (bytes / group_bytes) * units_per_group;  // whole row groups only
  const int64_t u0 = blockIdx.x * units / gridDim.x, u1 = (blockIdx.x + 1) * units / gridDim.x;
  if (warp == nw) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    for (int64_t u = u0; u < u1; ++u) {
      const int j = (int)(u - u0), s = j % stages;
      const uint32_t par = ((j / stages) & 1) ^ 1;
      asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(
                       sa(&empty[s])),
                   "r"(par));
      if (lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])),
                     "r"(stage_bytes));
      __syncwarp();
      const int64_t g = u / units_per_group, c = u % units_per_group;
      for (int r = lane; r < rows; r += 32) {
        const char* p = src + g * group_bytes + r * row_stride + c * piece;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, "
            "[%3], %4;" ::"r"(sa(sm + (size_t)s * stage_bytes + r * piece)),
            "l"(p), "r"(piece), "r"(sa(&full[s])), "l"(pol)
            : "memory");
      }
    }
    return;
  }
  float acc = 0.f;
  for (int64_t u = u0; u < u1; ++u) {
    const int j = (int)(u - u0), s = j % stages;
    const uint32_t par = (j / stages) & 1;
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(
                     sa(&full[s])),
                 "r"(par));
    const float4* st = reinterpret_cast<const float4*>(sm + (size_t)s * stage_bytes);
    for (int i = warp * 32 + lane; i < stage_bytes / 16; i += nw * 32) acc += st[i].x;
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])));
  }
  if (acc == 12345.f) *sink = acc;
}


__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, int64_t row_blocks, int kchunks, int stages,
                           int nbox, float* sink, const __grid_constant__ CUtensorMap xmap, int xbox) {
  extern __shared__ __align__(1024) unsigned char smraw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  const int stage_bytes = nbox * (16384 + xbox * 4096);  // xbox: + one 32 x 64 activation box per k-chunk (L2)
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + (size_t)stages * stage_bytes);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x / 32 - 1;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[s])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(&empty[s])), "r"(nw));
    }
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  const int per_unit = kchunks / nbox;
  const int64_t units = row_blocks * per_unit;
  const int64_t u0 = blockIdx.x * units / gridDim.x, u1 = (blockIdx.x + 1) * units / gridDim.x;
  if (warp == nw) {
    if (lane == 0) {
      for (int64_t u = u0; u < u1; ++u) {
        const int j = (int)(u - u0), s = j % stages;
        const uint32_t par = ((j / stages) & 1) ^ 1;
        asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(
                         sa(&empty[s])), "r"(par));
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(stage_bytes));
        const int64_t rb = u / per_unit;
        const int kc0 = (int)(u % per_unit) * nbox;
        for (int b = 0; b < nbox; ++b) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                  sa(sm + (size_t)s * stage_bytes + b * 16384)),
              "l"(&map), "r"(sa(&full[s])), "r"((kc0 + b) * 64), "r"((int)(rb * 128))
              : "memory");
          if (xbox)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                    sa(sm + (size_t)s * stage_bytes + nbox * 16384 + b * 4096)),
                "l"(&xmap), "r"(sa(&full[s])), "r"((kc0 + b) * 64), "r"(0)
                : "memory");
        }
      }
    }
    __syncwarp();
    return;
  }
  float acc = 0.f;
  for (int64_t u = u0; u < u1; ++u) {
    const int j = (int)(u - u0), s = j % stages;
    const uint32_t par = (j / stages) & 1;
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W;\n}" ::"r"(
                     sa(&full[s])), "r"(par));
    acc += reinterpret_cast<const float*>(sm + (size_t)s * stage_bytes)[threadIdx.x];
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])));
  }
  if (acc == 12345.f) *sink = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int U>
__global__ void ldg_kernel(const uint4* __restrict__ src, int64_t n16, float* sink) {
  float acc = 0.f;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(src + i + u * stride));
#pragma unroll
    for (int u = 0; u < U; ++u) acc += __uint_as_float(v[u].x ^ v[u].w);
  }
  if (acc == 12345.f) *sink = acc;
}

int main() {
  const int64_t bytes = 4LL << 30;  // 4 GiB per pass (>> L2)
  char* buf;
  float* sink;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&sink, 4);
  cudaMemset(buf, 1, bytes);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto timeit = [&](auto launch, const char* name) {
    for (int i = 0; i < 2; ++i) launch();
    cudaEventRecord(a);
    const int n = 5;
    for (int i = 0; i < n; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("%-52s %7.1f GB/s %s\n", name, bytes * n / (ms / 1e3) / 1e9, e ? cudaGetErrorString(e) : "");
  };
  struct Cfg { int stages, stage_kb, rows, row_kb, ctas; };
  Cfg cfgs[] = {{6, 32, 16, 8, 1},  {3, 64, 16, 8, 1}, {3, 64, 16, 28, 1}, {6, 32, 16, 28, 1},
                {3, 64, 1, 64, 1},  {3, 64, 8, 8, 1},  {2, 96, 16, 24, 1}, {4, 48, 16, 24, 1},
                {6, 32, 4, 8, 1},   {2, 112, 16, 28, 1}};
  for (auto c : cfgs) {
    const int stage_bytes = c.stage_kb * 1024;
    const int smem = c.stages * stage_bytes + 256;
    cudaFuncSetAttribute(bulk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    char name[128];
    snprintf(name, sizeof name, "bulk stages=%d stage=%dKiB rows=%d row_stride=%dKiB ctas/sm=%d", c.stages,
             stage_bytes / 1024, c.rows, c.row_kb, c.ctas);
    const int64_t rs = (int64_t)c.row_kb * 1024;
    timeit([&] { bulk_kernel<<<sms * c.ctas, 288, smem>>>(buf, bytes, c.stages, stage_bytes, c.rows, rs, sink); },
           name);
  }
  {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    EncodeFn enc = reinterpret_cast<EncodeFn>(fp);
    const int64_t K = 4096, rows = bytes / (K * 2);
    CUtensorMap map;
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)K * 2};
    cuuint32_t box[2] = {64, 128}, es[2] = {1, 1};
    for (int promo = 0; promo < 2; ++promo) {
      enc(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, promo ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B : CU_TENSOR_MAP_L2_PROMOTION_NONE,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      // x: a 32-row activation tensor (L2-resident), one 32 x 64 box per k-chunk when xbox
      CUtensorMap xmap;
      cuuint64_t xdims[2] = {(cuuint64_t)K, 32};
      cuuint32_t xb[2] = {64, 32};
      enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, xdims, strides, xb, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
          CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      struct T { int stages, nbox, xbox; } tc[] = {{12, 1, 0}, {6, 2, 0}, {3, 4, 0}, {4, 3, 0}, {3, 3, 0},
                                                   {3, 3, 1}, {2, 4, 1}, {5, 2, 1}, {10, 1, 1}};
      for (auto t : tc) {
        const int smem = t.stages * t.nbox * (16384 + t.xbox * 4096) + 1024 + 256;
        cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        char name[128];
        snprintf(name, sizeof name, "tma 128x64 SW128 boxes: %d stages x %d boxes%s promo=%d", t.stages, t.nbox,
                 t.xbox ? " (+x box each)" : "", promo);
        timeit([&] { tma_kernel<<<sms, 288, smem>>>(map, rows / 128, (int)(K / 64), t.stages, t.nbox, sink, xmap,
                                                     t.xbox); }, name);
      }
    }
  }
  timeit([&] { ldg_kernel<4><<<sms * 4, 256>>>((const uint4*)buf, bytes / 16, sink); }, "ldg v4 unroll4 4x256/sm");
  timeit([&] { ldg_kernel<8><<<sms * 4, 256>>>((const uint4*)buf, bytes / 16, sink); }, "ldg v4 unroll8 4x256/sm");
  timeit([&] { ldg_kernel<8><<<sms * 8, 256>>>((const uint4*)buf, bytes / 16, sink); }, "ldg v4 unroll8 8x256/sm");
  timeit([&] { cudaMemcpyAsync(buf + bytes / 2, buf, bytes / 2, cudaMemcpyDeviceToDevice); },
         "memcpy d2d (bytes = read+write)");
  const cudaError_t e = cudaDeviceSynchronize();
  if (e) printf("error: %s\n", cudaGetErrorString(e));
  return 0;
}
