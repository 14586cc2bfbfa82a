// Standalone probe: one 3-D tensor TMA load (fp64) into smem, compare with a plain copy.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstring>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int VARIANT>
__global__ void probe(const __grid_constant__ CUtensorMap map, double* out, int bx, int by, int c0, int c1, int c2) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* buf = reinterpret_cast<double*>(sm);
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bx * by * 8) : "memory");
    if (VARIANT == 0)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(smem_u32(buf)), "l"(&map), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(smem_u32(buf)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < bx * by; i += blockDim.x) out[i] = buf[i];
}

int main() {
  const int N = 32, bx = 24, by = 24;
  std::vector<double> h(N * N * N);
  for (int i = 0; i < N * N * N; ++i) h[i] = i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, bx * by * 8);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fp);
  CUtensorMap map;
  memset(&map, 0, sizeof(map));
  cuuint64_t dims[3] = {N, N, N}, strides[2] = {N * 8, N * N * 8};
  cuuint32_t box[3] = {bx, by, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d q %d\n", (int)r, (int)q);
  for (int v = 0; v < 2; ++v) {
    for (int c0 : {0, -3}) {
      cudaMemset(o, 0, bx * by * 8);
      if (v == 0) probe<0><<<1, 128, bx * by * 8>>>(map, o, bx, by, c0, -2, 5);
      else probe<1><<<1, 128, bx * by * 8>>>(map, o, bx, by, c0, -2, 5);
      cudaError_t e = cudaDeviceSynchronize();
      std::vector<double> ho(bx * by);
      cudaMemcpy(ho.data(), o, bx * by * 8, cudaMemcpyDeviceToHost);
      int bad = 0;
      for (int y = 0; y < by; ++y)
        for (int x = 0; x < bx; ++x) {
          int gx = c0 + x, gy = -2 + y;
          double ex = (gx >= 0 && gx < N && gy >= 0 && gy < N) ? h[(5 * N + gy) * N + gx] : 0.0;
          if (ho[y * bx + x] != ex) bad++;
        }
      printf("variant %d c0 %d: %s bad=%d\n", v, c0, cudaGetErrorString(e), bad);
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
