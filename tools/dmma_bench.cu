// Is the FP64 tensor core (DMMA, mma.sync m8n8k4 f64) a separate pipe from the FP64 CUDA-core
// pipe on sm_100a?  Times DFMA-only, DMMA-only and mixed streams.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}

template <int NF, int NM>
__global__ void __launch_bounds__(256) k(double* out, int iters, const double* __restrict__ init) {
  double x[8], m[8];
  double acc[4][2];
  double a = init[threadIdx.x % 64], b = init[64 + threadIdx.x % 64];
#pragma unroll
  for (int i = 0; i < 8; ++i) { x[i] = init[(threadIdx.x + i) % 128]; m[i] = init[(threadIdx.x * 3 + i) % 128]; }
#pragma unroll
  for (int i = 0; i < 4; ++i) { acc[i][0] = 0; acc[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
#pragma unroll
      for (int i = 0; i < NF; ++i)
        asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(x[i & 7]) : "d"(m[i & 7]));
#pragma unroll
      for (int j = 0; j < NM; ++j) dmma(acc[j & 3], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
  if (s == 1234.5) out[0] = s;
}

template <int NF, int NM>
void run(double* d, const char* name) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 4, iters = 4096;
  k<NF, NM><<<blocks, 256>>>(d, 16, d + 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k<NF, NM><<<blocks, 256>>>(d, iters, d + 8);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double warps = blocks * 8.0;
  const double dfma_lane_ops = warps * 32 * iters * 4.0 * NF;
  const double dmma_macs = warps * iters * 4.0 * NM * 256;
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("%-14s %8.3f ms  DFMA %.1f lane-FMA/clk/SM  DMMA %.1f MAC/clk/SM  total %.1f\n", name, ms,
         dfma_lane_ops / cyc / sms, dmma_macs / cyc / sms, (dfma_lane_ops + dmma_macs) / cyc / sms);
}

int main() {
  double* d;
  cudaMalloc(&d, 8 * 256);
  double h[256];
  for (int i = 0; i < 256; ++i) h[i] = 0.999 + 1e-6 * i;
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  run<8, 0>(d, "dfma only");
  run<0, 4>(d, "dmma only");
  run<8, 1>(d, "8 dfma+1 dmma");
  run<8, 2>(d, "8 dfma+2 dmma");
  run<8, 4>(d, "8 dfma+4 dmma");
  return 0;
}
