// Kernel-boundary cost probe (development aid): a chain of dependent small
// kernels launched plainly vs with programmatic dependent launch (PDL).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pdl_probe tools/pdl_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_step(float* buf, int n, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (pdl == 2) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) buf[i] = buf[i] * 1.0001f + 1.f;
}

int main() {
  const int n = 148 * 256 * 4;
  float* buf;
  cudaMalloc(&buf, n * sizeof(float));
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int grid : {148, 592}) {
    for (int pdl = 0; pdl < 3; ++pdl) {
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(256);
      cfg.stream = s;
      cfg.attrs = pdl ? at : nullptr;
      cfg.numAttrs = pdl ? 1 : 0;
      const int m = grid * 256;
      const int K = 2000;
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
      for (int k = 0; k < K; ++k) cudaLaunchKernelEx(&cfg, k_step, buf, m, pdl);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, s);
        if (rep == 2) {
          for (int k = 0; k < K; ++k) cudaLaunchKernelEx(&cfg, k_step, buf, m, pdl);
        } else {
          cudaGraphLaunch(ge, s);
        }
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("grid %d pdl %d %s: %.3f us per kernel\n", grid, pdl, rep == 2 ? "stream" : "graph", 1e3f * ms / K);
      }
    }
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
