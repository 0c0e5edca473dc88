// TMA bulk-copy (cp.async.bulk global -> shared, mbarrier complete_tx) throughput per SM:
// one CTA per SM streams CHUNK-byte copies through a STAGES-deep ring (one elected thread
// issues, every copy completes on its stage's mbarrier; the same thread waits and re-issues).
// Modes: 0 = every CTA reads its own region, 1 = all CTAs read the same SPAN bytes,
// 2 = CTAs read overlapping windows (CTA b starts at b * 16 KB mod SPAN).
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/tma_bench tools/tma_bench.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }

__global__ void tma_kernel(const char* src, size_t span, int chunk, int stages, int iters, int mode,
                           unsigned long long* cyc) {
  extern __shared__ __align__(128) unsigned char sm[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + size_t(stages) * chunk);
  if (threadIdx.x != 0) return;
  for (int s = 0; s < stages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t base = mode == 0 ? size_t(blockIdx.x) * span : (mode == 2 ? (size_t(blockIdx.x) * 16384) % span : 0);
  const size_t region = span;
  auto issue = [&](int f) {
    const int s = f % stages;
    const size_t off = (mode == 0 ? base : 0) + ((mode == 2 ? base : 0) + size_t(f) * chunk) % region;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar[s])), "r"(chunk) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                     "r"(su32(sm + size_t(s) * chunk)), "l"(src + off), "r"(chunk), "r"(su32(&bar[s])) : "memory");
  };
  const long long t0 = clock64();
  for (int f = 0; f < stages && f < iters; ++f) issue(f);
  for (int f = 0; f < iters; ++f) {
    const int s = f % stages;
    const uint32_t par = (f / stages) & 1;
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(su32(&bar[s])), "r"(par) : "memory");
    if (f + stages < iters) issue(f + stages);
  }
  cyc[blockIdx.x] = clock64() - t0;
}

int main(int argc, char** argv) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = size_t(1) << 31;  // 2 GB source
  char* src;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * 1024);
  cudaFuncSetAttribute(tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  struct Case { int mode; size_t span; int chunk, stages, grid; } cases[] = {
      {0, 8 << 20, 16384, 4, sms}, {0, 8 << 20, 16384, 8, sms}, {0, 8 << 20, 4096, 16, sms},
      {0, 8 << 20, 32768, 4, sms}, {1, 65536, 16384, 4, sms}, {1, 1 << 20, 16384, 4, sms},
      {2, 1 << 20, 16384, 4, sms}, {2, 8 << 20, 16384, 4, sms}, {0, 8 << 20, 16384, 4, 1},
      {1, 65536, 16384, 4, 1}};
  if (argc > 1) {  // L2 sharing probe: every CTA streams the same SPAN once (ncu: DRAM bytes)
    const size_t span = size_t(atoi(argv[1])) << 20;
    const int iters = int(span / 16384);
    const int mode = argc > 2 ? atoi(argv[2]) : 1;
    tma_kernel<<<sms, 32, 4 * 16384 + 32>>>(src, span, 16384, 4, iters, mode, cyc);
    cudaDeviceSynchronize();
    printf("probe span %zu MB x %d CTAs\n", span >> 20, sms);
    return 0;
  }
  for (auto& c : cases) {
    const int iters = 2000;
    const size_t smem = size_t(c.stages) * c.chunk + 8 * c.stages;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    tma_kernel<<<c.grid, 32, smem>>>(src, c.span, c.chunk, c.stages, 50, c.mode, cyc);
    cudaEventRecord(e0);
    tma_kernel<<<c.grid, 32, smem>>>(src, c.span, c.chunk, c.stages, iters, c.mode, cyc);
    cudaEventRecord(e1);
    cudaError_t e = cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(c.grid) * iters * c.chunk;
    printf("mode %d span %8zu chunk %6d stages %2d grid %3d: %8.3f ms  total %8.1f GB/s  per SM %7.1f GB/s  %s\n",
           c.mode, c.span, c.chunk, c.stages, c.grid, ms, bytes / ms / 1e6, bytes / ms / 1e6 / c.grid,
           cudaGetErrorString(e));
  }
  return 0;
}
