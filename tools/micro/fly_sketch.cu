// Measured A/B for SURVEY 8(a) A4 "sketch each new column in the same pass that produces it": the per-column cost
// of applying the hashed sparse sign map ON THE FLY (hash the row's zeta = 8 (row, sign) pairs, scatter-add into a
// per-CTA shared-memory s-vector, per-CTA partials reduced afterwards) -- the work an in-pass sketch would add to
// the step kernel -- against the batched plan + gather sketch the library uses (17.6 us per column at J = 32, C3).
// Variants: (hash) hashing only, no accumulation; (atomic) + fp64 shared-memory atomicAdd (CAS loops on sm_100a).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2111_00113_b200/csrc fly_sketch.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "common.cuh"

template <int MODE>
__global__ void __launch_bounds__(512) fly_kernel(const double* __restrict__ w, int64_t n, int s, uint64_t key,
                                                  double* __restrict__ part, double* __restrict__ sink) {
  extern __shared__ double acc[];
  for (int i = threadIdx.x; i < s; i += blockDim.x) acc[i] = 0.0;
  __syncthreads();
  const double sc = 1.0 / sqrt(8.0);
  double dummy = 0.0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const double v = w[r] * sc;
    int q[8];
    uint32_t neg;
    sks_column_rt(key, (uint64_t)r, s, 8, q, &neg);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      const double x = ((neg >> t) & 1u) ? -v : v;
      if (MODE == 1) atomicAdd(&acc[q[t]], x);
      else dummy += x * (double)q[t];
    }
  }
  __syncthreads();
  if (MODE == 0 && dummy == 12345.678) sink[0] = dummy;
  for (int i = threadIdx.x; i < s; i += blockDim.x) part[(int64_t)blockIdx.x * s + i] = acc[i];
}

int main() {
  const int64_t n = 4096000;  // C3
  const int s = 600;
  double *w, *part, *sink;
  cudaMalloc(&w, n * 8);
  cudaMalloc(&part, 148 * 4 * s * 8);
  cudaMalloc(&sink, 8);
  cudaMemset(w, 0, n * 8);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int mode = 0; mode < 2; ++mode) {
    for (int cps : {1, 2, 4}) {
      const int grid = sms * cps;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        for (int it = 0; it < 20; ++it) {
          if (mode == 0) fly_kernel<0><<<grid, 512, s * 8>>>(w, n, s, 0x1234567ull + it, part, sink);
          else fly_kernel<1><<<grid, 512, s * 8>>>(w, n, s, 0x1234567ull + it, part, sink);
        }
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("%s ctas/SM=%d: %.1f us per column (n = %lld, s = %d, zeta = 8)\n",
                        mode ? "hash + fp64 smem atomicAdd" : "hash only", cps, ms * 1000 / 20, (long long)n, s);
      }
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
