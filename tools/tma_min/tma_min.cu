// Minimal TMA probe: which descriptor placement / instruction form works on this box.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include "../../paper_2111_00113_b200/csrc/tma.cuh"

__global__ void k_param(const __grid_constant__ CUtensorMap tm, double* out, int mode) {
  __shared__ __align__(128) double buf[36 * 12];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    if (mode >= 1) tma_prefetch_desc(&tm);
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (mode >= 2) {
    if (threadIdx.x == 0) {
      mbar_arrive_expect_tx(&bar, 36 * 12 * 8);
      tma_load_3d(buf, &tm, &bar, -2, 0, 0);
    }
    mbar_wait(&bar, 0);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 36 * 12; i += blockDim.x) out[i] = buf[i];
}

__global__ void k_global(const CUtensorMap* tm, double* out) {
  __shared__ __align__(128) double buf[36 * 12];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_arrive_expect_tx(&bar, 36 * 12 * 8);
    tma_load_3d(buf, tm, &bar, -2, 0, 0);
  }
  mbar_wait(&bar, 0);
  __syncthreads();
  for (int i = threadIdx.x; i < 36 * 12; i += blockDim.x) out[i] = buf[i];
}

int main(int argc, char** argv) {
  int mode = atoi(argv[1]);
  const int m = 32, ny = 20, nc = 3;
  double* g;
  cudaMalloc(&g, sizeof(double) * m * ny * nc);
  double h[m * ny * nc];
  for (int i = 0; i < m * ny * nc; ++i) h[i] = i;
  cudaMemcpy(g, h, sizeof(h), cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, sizeof(double) * 36 * 12);
  cudaMemset(out, 0, sizeof(double) * 36 * 12);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  CUtensorMap tm;
  cuuint64_t dims[3] = {m, ny, nc};
  cuuint64_t str[2] = {m * 8, (cuuint64_t)m * ny * 8};
  cuuint32_t box[3] = {36, 12, 1}, es[3] = {1, 1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, g, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode=%d fn=%p q=%d\n", (int)r, fn, (int)q);
  if (mode < 3) {
    k_param<<<1, 128>>>(tm, out, mode);
  } else {
    CUtensorMap* dtm;
    cudaMalloc(&dtm, sizeof(CUtensorMap));
    cudaMemcpy(dtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
    k_global<<<1, 128>>>(dtm, out);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("mode %d: %s\n", mode, cudaGetErrorString(e));
  double ho[36 * 12];
  cudaMemcpy(ho, out, sizeof(ho), cudaMemcpyDeviceToHost);
  printf("row0: %g %g %g %g ... row1 x2: %g  (expect 0 0 0 1 ... 32)\n", ho[0], ho[1], ho[2], ho[3], ho[36 + 2]);
  return 0;
}
