// Micro-probe: cost of cluster barriers and dependent global round trips inside one
// 8-CTA cluster (B200).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

struct Big { int n; double pad[1000]; };

__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024, 1) k_sync(int n, double* buf) {
  cg::cluster_group cl = cg::this_cluster();
  for (int i = 0; i < n; ++i) cl.sync();
}
__global__ void __cluster_dims__(8, 1, 1) __launch_bounds__(1024, 1) k_ld_sync(int n, double* buf, int cells) {
  cg::cluster_group cl = cg::this_cluster();
  const int tid = cl.block_rank() * 1024 + threadIdx.x;
  for (int i = 0; i < n; ++i) {
    for (int c = tid; c < cells; c += 8192) buf[c] = buf[c] * 0.5 + 1.0;
    cl.sync();
  }
}
__global__ void __launch_bounds__(1024, 1) k_cta(int n, double* buf, int cells) {
  for (int i = 0; i < n; ++i) {
    for (int c = threadIdx.x; c < cells; c += 1024) buf[c] = buf[c] * 0.5 + 1.0;
    __syncthreads();
  }
}
__global__ void k_big(const __grid_constant__ Big b, double* out) { if (threadIdx.x == 0) out[0] = b.pad[b.n]; }
__global__ void k_small(int n, double* out) { if (threadIdx.x == 0) out[0] = n; }

int main() {
  double* buf;
  cudaMalloc(&buf, 64 << 20);
  cudaMemset(buf, 0, 64 << 20);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  auto T = [&](const char* name, auto f, int reps) {
    f();
    cudaDeviceSynchronize();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %9.3f us per call  (%s)\n", name, 1e3 * ms / reps, cudaGetErrorString(cudaGetLastError()));
  };
  T("k_sync n=0", [&] { k_sync<<<8, 1024>>>(0, buf); }, 100);
  T("k_sync n=100", [&] { k_sync<<<8, 1024>>>(100, buf); }, 100);
  T("k_ld_sync n=100 cells=512", [&] { k_ld_sync<<<8, 1024>>>(100, buf, 512); }, 100);
  T("k_ld_sync n=100 cells=32768", [&] { k_ld_sync<<<8, 1024>>>(100, buf, 32768); }, 100);
  T("k_cta n=100 cells=512", [&] { k_cta<<<1, 1024>>>(100, buf, 512); }, 100);
  T("k_cta n=100 cells=4096", [&] { k_cta<<<1, 1024>>>(100, buf, 4096); }, 100);
  T("k_cta n=100 cells=32768", [&] { k_cta<<<1, 1024>>>(100, buf, 32768); }, 100);
  Big big{};
  big.n = 3;
  T("k_big (8 KB param)", [&] { k_big<<<1, 32>>>(big, buf); }, 1000);
  T("k_small", [&] { k_small<<<1, 32>>>(3, buf); }, 1000);
  return 0;
}
