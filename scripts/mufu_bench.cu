// MUFU ex2 throughput microbenchmark ("Verify the MUFU rate with a
// microbenchmark").  Every thread runs 8 independent chains of ex2.approx.ftz.f32; the kernel
// time gives ex2 / s per GPU, compared with 148 SM x 16 / clk x f_SM.  Tooling, not product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_bench scripts/mufu_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ex2(float* out, int iters) {
  float v[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) v[u] = 1e-3f * (threadIdx.x + u);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      float r;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(v[u]));
      v[u] = r * -0.5f;                       // keeps the chain bounded (|v| < 1)
    }
  }
  float s = 0.f;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += v[u];
  if (s == 12345.f) out[0] = s;               // defeat dead-code elimination
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  const int iters = 4096, threads = 512, blocks = sms * 4;
  k_ex2<<<blocks, threads>>>(out, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(a);
    k_ex2<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  const double n = (double)blocks * threads * iters * 8;
  const double rate = n / (best * 1e-3);
  printf("{\"ex2_per_s\": %.4g, \"sms\": %d, \"clock_mhz_attr\": %.0f, \"ex2_per_clk_per_sm_at_attr_clock\": %.2f, "
         "\"ms\": %.3f}\n", rate, sms, clk_khz / 1e3, rate / (sms * clk_khz * 1e3), best);
  return 0;
}
