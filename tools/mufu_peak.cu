// MUFU.EX2 throughput probe: the second pipe the compositing kernels lean
// on (one ex2.approx per evaluated (pixel, entry) pair).  8 independent
// ex2 chains per thread, 148 x 8 CTAs x 256 threads, best of 10.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void k_ex2(float* out, int iters) {
  float x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = -0.001f * (threadIdx.x + k);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = ex2(x[k]) - 1.0f;  // stays in (-1, 0]
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 1024;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ex2<<<blocks, threads>>>(out, 16);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_ex2<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = 8.0 * 16 * (double)iters * blocks * threads;
  const double per_sm_clk = ops / (best * 1e-3) / sms / (clk * 1e3);
  printf("{\"ex2_gops\": %.1f, \"ex2_per_sm_per_clk\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f, "
         "\"how\": \"8 independent ex2.approx.ftz chains (+1 FADD each)/thread, %d CTAs x %d threads, best of 10\"}\n",
         ops / (best * 1e-3) / 1e9, per_sm_clk, sms, clk / 1e3, blocks, threads);
  return 0;
}
