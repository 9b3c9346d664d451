// FP32 FFMA throughput probe (the roofline denominator for the FP32-pipe
// bound compositing kernels; MEASURED_PEAKS.json only carries HBM and bf16).
// 8 independent FFMA chains per thread, 148 x 8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_ffma(float* out, int iters, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
      x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  float* out;
  cudaMalloc(&out, sizeof(float) * blocks * threads);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ffma<<<blocks, threads>>>(out, 64, 0.999f, 0.001f);
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0);
    k_ffma<<<blocks, threads>>>(out, iters, 0.999f, 0.001f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf("{\"fp32_tflops\": %.2f, \"sms\": %d, \"max_clock_mhz\": %.0f, \"nominal_tflops\": %.2f, "
         "\"how\": \"8 independent FFMA chains/thread, %d CTAs x %d threads, best of 10, CUDA events\"}\n",
         flops / (best * 1e-3) / 1e12, sms, clk / 1e3, 2.0 * 128 * sms * clk * 1e3 / 1e12, blocks, threads);
  return 0;
}
