// TMA 1D box test (diagnostics)
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdint>
#include "../../paper_2310_14712_b200/csrc/explicit_common.cuh"
#include "../../paper_2310_14712_b200/csrc/explicit3d.cuh"
#include "../../paper_2310_14712_b200/csrc/explicit3d_xyz.cuh"
__global__ void k(const __grid_constant__ CUtensorMap map, double* out, int x0, int mode) {
  extern __shared__ __align__(128) double sm[];
  __shared__ uint64_t bar[1];
  if (threadIdx.x == 0) xyz::mbar_init(&bar[0]);
  __syncthreads();
  if (threadIdx.x == 0) {
    xyz::mbar_expect(&bar[0], 2 * 32 * 8);
    xyz::tma_row(sm, &map, x0, &bar[0]);
    xyz::tma_row(sm + 32, &map, x0 + 1000, &bar[0]);
  }
  xyz::mbar_wait(&bar[0], 0);
  out[threadIdx.x] = sm[threadIdx.x];
  out[32 + threadIdx.x] = sm[32 + threadIdx.x];
}
int main() {
  const size_t n = 1 << 20;
  double* a; double* o;
  cudaMalloc(&a, n * 8); cudaMalloc(&o, 64 * 8);
  double* h = new double[n];
  for (size_t i = 0; i < n; ++i) h[i] = (double)i;
  cudaMemcpy(a, h, n * 8, cudaMemcpyHostToDevice);
  PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
  CUtensorMap map;
  const cuuint64_t dims[1] = {n};
  const cuuint64_t strides[1] = {8};
  const cuuint32_t box[1] = {32};
  const cuuint32_t es[1] = {1};
  CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 1, (void*)a, dims, strides, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d\n", (int)r);
  for (int x0 : {0, 5, -3}) {
    k<<<1, 32, 1024>>>(map, o, x0, 0);
    cudaError_t e = cudaDeviceSynchronize();
    printf("x0=%d: %s\n", x0, cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    double ho[64];
    cudaMemcpy(ho, o, 64 * 8, cudaMemcpyDeviceToHost);
    printf("  %g %g %g ... %g %g\n", ho[0], ho[1], ho[31], ho[32], ho[63]);
  }
  return 0;
}
