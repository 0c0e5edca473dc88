// FP64 issue-rate microbenchmark: does a DFMA with three distinct, non-reused register
// sources issue slower than one with two?  (register-file read model, B300_MICROARCH.md)
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(256) k(double* out, int iters, const double* __restrict__ init) {
  double x[8], m[8], c[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    x[i] = init[(threadIdx.x * 24 + i) % 4096];
    m[i] = init[(threadIdx.x * 24 + 8 + i) % 4096];
    c[i] = init[(threadIdx.x * 24 + 16 + i) % 4096];
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0)  // 3 distinct per-chain registers
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(m[i]), "d"(c[i]));
        if (MODE == 1)  // shared operands (reuse cache)
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(m[0]), "d"(c[0]));
        if (MODE == 2)  // 2 distinct
          asm volatile("fma.rn.f64 %0, %0, %1, %0;" : "+d"(x[i]) : "d"(m[i]));
        if (MODE == 3) asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(x[i]) : "d"(m[i]));
        if (MODE == 4) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(x[i]) : "d"(c[i]));
        if (MODE == 5)  // 3 distinct, one shared with the previous instruction (slot B)
          asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(x[i]) : "d"(m[0]), "d"(c[i]));
      }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 1234.5) out[0] = s;
}

template <int MODE>
float run(double* d, int blocks) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<MODE><<<blocks, 256>>>(d, 64, d + 1);
  cudaEventRecord(a);
  const int iters = 2048;
  k<MODE><<<blocks, 256>>>(d, iters, d + 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double warp_instr = double(blocks) * 8 * iters * 64;
  double per_smsp_cycles = ms * 1e-3 * clk * 1e3;
  double ipc = warp_instr / (sms * 4) / per_smsp_cycles;
  printf("mode %d: %.3f ms, %.3f DP warp-instr/cycle/SMSP (peak 0.5)\n", MODE, ms, ipc);
  return ms;
}

int main() {
  double* d;
  cudaMalloc(&d, 8 * 4200);
  double h[4200];
  for (int i = 0; i < 4200; ++i) h[i] = (i % 3 == 0) ? 0.9999999 : 1e-9 * (i % 97);
  cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int occ : {2, 4}) {
    printf("blocks per SM %d\n", occ);
    run<0>(d, sms * occ);
    run<1>(d, sms * occ);
    run<2>(d, sms * occ);
    run<3>(d, sms * occ);
    run<4>(d, sms * occ);
    run<5>(d, sms * occ);
  }
  return 0;
}
