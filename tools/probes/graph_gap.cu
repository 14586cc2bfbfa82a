// Per-node overhead of a CUDA graph of dependent kernels on this GPU: a chain of N tiny
// kernels (one CTA each, and 148x2 CTAs each), captured once and replayed.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_tiny(float* p) { if (threadIdx.x == 0) p[blockIdx.x] += 1.0f; }
int main() {
  float* d;
  cudaMalloc(&d, 4096 * sizeof(float));
  cudaStream_t s;
  cudaStreamCreate(&s);
  for (int grid : {1, 296}) {
    for (int n : {1, 56, 200}) {
      cudaGraph_t g;
      cudaGraphExec_t ge;
      cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      for (int i = 0; i < n; ++i) k_tiny<<<grid, 256, 0, s>>>(d);
      cudaStreamEndCapture(s, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int w = 0; w < 5; ++w) cudaGraphLaunch(ge, s);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, s);
      const int reps = 50;
      for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      printf("grid %4d  nodes %4d  %.2f us per graph  %.3f us per node\n", grid, n,
             ms * 1e3 / reps, ms * 1e3 / reps / n);
    }
  }
  return 0;
}
