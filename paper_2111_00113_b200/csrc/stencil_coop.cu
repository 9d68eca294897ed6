// stencil_coop.cu -- a whole batch of truncated-Arnoldi / Chebyshev columns in ONE cooperative launch, for small
// stencil problems (C1, C2: vectors of a few MB that live in L2) where a column's work is a few microseconds and
// the per-launch chain of the persistent step kernels (prologue reduction, TMA pipeline fill, epilogue, launch
// gap: ~14 us at C2) dominates.  Single rank only (a grid barrier replaces the per-column halo exchange and
// all-reduce).
//
// Per column j (Eq. partorth P:208-218 / Eq. Chebrecurse, the same arithmetic as step.cuh):
//   every CTA re-reduces the previous column's per-CTA partials in a fixed order (step_prologue: identical
//   coefficients in every CTA, bookkeeping by CTA 0), forms w_j = alpha A u + beta u + sum c_l V_l on its share
//   of the rows (neighbours through L1/L2), grid barrier, then the partial sums the next column needs
//   (||w_j||^2, <w_j, A w_j>, ||A w_j||^2, <V_l, A w_j>, <u, A w_j>; step_epilogue's slots), grid barrier.
// The partials use the same ping-pong slots as the per-column kernels, so batches and single launches mix.
#include "common.cuh"
#include "internal.h"
#include "step.cuh"

namespace sks {

constexpr int CO_T = 512;

struct CoopArgs {
  StepArgs a;       // geometry, recurrence state; a.j / partials set per column inside the kernel
  int j0, j1;       // columns [j0, j1]
  int grid_prev0;   // rows of the partials of column j0 - 1
  double* part;     // ping-pong partial slots: slot (j & 1) at part + (j & 1) * pstride * SKS_NP
  int pstride;
  unsigned* sync;   // grid barrier: [0] count, [1] generation (zero at launch)
};

__device__ __forceinline__ void co_grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(const_cast<unsigned*>(gen), 1u);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ double co_apply(const double* __restrict__ u, int64_t idx, int64_t plane, int64_t m,
                                           int dim, double cc, double cm, double cp) {
  const int64_t z = idx / plane, ip = idx - z * plane;
  const int64_t x = (dim == 3) ? ip % m : ip, y = (dim == 3) ? ip / m : 0;
  const double* p = u + idx;
  double sm = p[-plane] + (x > 0 ? p[-1] : 0.0);  // ghost planes hold the Dirichlet zeros
  double sp = p[plane] + (x < m - 1 ? p[1] : 0.0);
  if (dim == 3) {
    sm += (y > 0) ? p[-m] : 0.0;
    sp += (y < m - 1) ? p[m] : 0.0;
  }
  return cc * p[0] + cm * sm + cp * sp;
}

template <int KM>
__global__ void __launch_bounds__(CO_T) step_coop_kernel(CoopArgs ca) {
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  StepArgs a = ca.a;
  const int64_t n = a.nz * a.plane;
  const int64_t tid0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, tstride = (int64_t)gridDim.x * blockDim.x;
  for (int j = ca.j0; j <= ca.j1; ++j) {
    a.j = j;
    a.mode = 0;
    a.partials_in = ca.part + (size_t)((j - 1) & 1) * ca.pstride * SKS_NP;
    a.grid_prev = (j == ca.j0) ? ca.grid_prev0 : (int)gridDim.x;
    a.partials_out = ca.part + (size_t)(j & 1) * ca.pstride * SKS_NP;
    if (!step_prologue(a, &cf, red)) return;  // breakdown / early exit: uniform over the grid (same data)
    const double* U = cf.U + a.off;
    double* Wj = a.W + (int64_t)j * a.ld + a.off;
    const int nv = cf.nv;
    // ---- w_j on this CTA's rows
    for (int64_t r = tid0; r < n; r += tstride) {
      double w = cf.alpha * co_apply(U, r, a.plane, a.m, a.dim, a.cc, a.cm, a.cp) + cf.beta_u * U[r];
#pragma unroll
      for (int l = 0; l < KM - 1; ++l)
        if (l < nv) w += cf.c[l] * cf.V[l][a.off + r];
      Wj[r] = w;
    }
    co_grid_barrier(ca.sync, ca.sync + 1, gridDim.x);
    // ---- the next column's partial sums
    double acc[KM + 3];
#pragma unroll
    for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;
    for (int64_t r = tid0; r < n; r += tstride) {
      const double w = Wj[r];
      const double Aw = co_apply(Wj, r, a.plane, a.m, a.dim, a.cc, a.cm, a.cp);
      acc[0] = fma(w, w, acc[0]);
      acc[1] = fma(w, Aw, acc[1]);
      acc[2] = fma(Aw, Aw, acc[2]);
#pragma unroll
      for (int l = 0; l < KM - 1; ++l)
        if (l < nv && cf.vslot[l] >= 0) acc[3 + l] = fma(cf.V[l][a.off + r], Aw, acc[3 + l]);
      if (cf.uslot >= 0) acc[KM + 2] = fma(U[r], Aw, acc[KM + 2]);
    }
    step_epilogue<KM>(a, &cf, acc, red);
    co_grid_barrier(ca.sync, ca.sync + 1, gridDim.x);
  }
}

int coop_grid(int main_sms) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, step_coop_kernel<4>, CO_T, 0) != cudaSuccess || per < 1) {
    cudaGetLastError();
    return 0;
  }
  return main_sms * std::min(per, 1);
}

cudaError_t launch_step_coop(const StepArgs& a, int j0, int j1, int grid_prev0, double* part, int pstride,
                             unsigned* sync, int grid, cudaStream_t st) {
  CoopArgs ca;
  ca.a = a;
  ca.j0 = j0;
  ca.j1 = j1;
  ca.grid_prev0 = grid_prev0;
  ca.part = part;
  ca.pstride = pstride;
  ca.sync = sync;
  cudaError_t e = cudaMemsetAsync(sync, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&ca};
  const void* fn;
  switch (step_km(a.k)) {
    case 2: fn = (const void*)step_coop_kernel<2>; break;
    case 4: fn = (const void*)step_coop_kernel<4>; break;
    default: fn = (const void*)step_coop_kernel<8>; break;
  }
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(CO_T), args, 0, st);
}

// the batch runs against a private copy of the control block with exit_cols cleared (the side stream's sketched
// QR may set the real one at any time; every CTA must take the same decisions), merged back afterwards
__global__ void ctrl_copy_kernel(CtrlBlock* dst, const CtrlBlock* src) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    *dst = *src;
    dst->exit_cols = 0;
  }
}
__global__ void ctrl_merge_kernel(CtrlBlock* real, const CtrlBlock* priv, int first) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    if (priv->stop_col < real->stop_col) real->stop_col = priv->stop_col;
    if (priv->breakdown) real->breakdown = 1;
    if (first) real->rnorm = priv->rnorm;
  }
}

cudaError_t launch_ctrl_copy(CtrlBlock* dst, const CtrlBlock* src, cudaStream_t st) {
  ctrl_copy_kernel<<<1, 32, 0, st>>>(dst, src);
  return cudaGetLastError();
}
cudaError_t launch_ctrl_merge(CtrlBlock* real, const CtrlBlock* priv, int first, cudaStream_t st) {
  ctrl_merge_kernel<<<1, 32, 0, st>>>(real, priv, first);
  return cudaGetLastError();
}

}  // namespace sks
