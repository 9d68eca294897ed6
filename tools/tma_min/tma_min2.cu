// Probe: U box {68,36,1} + V box {66,34,1} on a {32, 36, 10} tensor, two loads, one barrier.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../../paper_2111_00113_b200/csrc/tma.cuh"

__global__ void k(const __grid_constant__ CUtensorMap tu, const __grid_constant__ CUtensorMap tv, double* out, int mode, int xv, int bvx) {
  extern __shared__ __align__(128) unsigned char raw[];
  double* s = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t bytes = 68 * 36 * 8 + (mode >= 1 ? bvx * 34 * 8 : 0);
    mbar_arrive_expect_tx(&bar, bytes);
    tma_load_3d(s, &tu, &bar, -2, 0, 1);
    if (mode >= 1) tma_load_3d(s + 2448, &tv, &bar, xv, 1, 1);
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  for (int i = threadIdx.x; i < 2448 + 2256; i += blockDim.x) out[i] = s[i];
}

int main(int argc, char** argv) {
  int mode = atoi(argv[1]); int xv = atoi(argv[2]); int bvx = atoi(argv[3]);
  const int m = 32, ny = 36, nc = 10;
  double* g;
  cudaMalloc(&g, sizeof(double) * m * ny * nc);
  double* h = (double*)malloc(sizeof(double) * m * ny * nc);
  for (int i = 0; i < m * ny * nc; ++i) h[i] = i;
  cudaMemcpy(g, h, sizeof(double) * m * ny * nc, cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, sizeof(double) * 4704);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tu, tv;
  cuuint64_t dims[3] = {m, ny, nc};
  cuuint64_t str[2] = {m * 8, (cuuint64_t)m * ny * 8};
  cuuint32_t bu[3] = {68, 36, 1}, bv[3] = {(cuuint32_t)bvx, 34, 1}, es[3] = {1, 1, 1};
  CUresult r1 = enc(&tu, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, bu, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  CUresult r2 = enc(&tv, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, bv, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode %d %d\n", (int)r1, (int)r2);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  k<<<1, 256, 40000>>>(tu, tv, out, mode, xv, bvx);
  cudaError_t e = cudaDeviceSynchronize();
  printf("xv %d bvx %d: %s\n", xv, bvx, cudaGetErrorString(e));
  double ho[4704];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("U[0,2]=%g (exp %d)  V[0,1]=%g (exp %d)\n", ho[2], 32 * 36, ho[2448 + 1], 32 * 36 * (mode == 2 ? 2 : 1) + 32);
  return 0;
}
