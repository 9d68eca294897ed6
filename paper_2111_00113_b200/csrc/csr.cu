// csr.cu -- truncated-Arnoldi step for a general sparse A in CSR (config C4).
//
// A general sparse A needs the whole of b_{j-1} before any row of A b_{j-1} is known,
// so one column takes two launches:
//   spmv_dots(j):  mr = A w_{j-1} (unscaled), stored;  partials ||mr||^2, <w_i, mr>
//                  for the window i = max(0,j-k) .. j-1 (classical GS, reading O8);
//   orth(j):       sigma_{j-1} = 1/||w_{j-1}||, h_i = sigma_{j-1} sigma_i <w_i, mr>,
//                  w_j = sigma_{j-1} mr - sum_i h_i sigma_i w_i;  partial ||w_j||^2.
// (Eq. partorth; Alg. 1.)  Per-CTA partials are re-reduced in a
// fixed order by every CTA of the next launch (deterministic, no atomics).
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace sks {

constexpr int CSR_G = 8;  // lanes per row

struct CsrArgs {
  int64_t n;            // local rows
  const int32_t* rp;    // local row_ptr (n+1)
  const int32_t* ci;    // column indices into the gathered vector xg
  const double* va;
  const double* xg;     // vector multiplied (w_{j-1}, or x for the residual)
  double* out;          // mr (spmv) / r (residual)
  const double* f;      // residual: f
  int mode;             // 0: spmv+dots, 1: residual r = f - A x
  // dots
  const double* W;      // basis columns, pitch ld
  int64_t ld;
  int lo, nw;           // window [lo, lo+nw)
  double* partials;     // [grid][SKS_NP]
  const CtrlBlock* ctrl; // may be NULL; early exit -> no-op
};

template <int KM>
__global__ void __launch_bounds__(256) csr_spmv_kernel(CsrArgs a) {
  __shared__ double red[SKS_NP * 32];
  const int tid = threadIdx.x;
  if (a.ctrl && (a.ctrl->exit_cols != 0 || a.ctrl->stop_col < 0x7fffffff)) return;
  const int sub = tid & (CSR_G - 1);
  const int grp = (tid & 31) / CSR_G;  // row group inside the warp
  constexpr int RPW = 32 / CSR_G;      // rows per warp step
  const int64_t wglob = (blockIdx.x * (int64_t)blockDim.x + tid) >> 5;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc[KM + 1];
#pragma unroll
  for (int i = 0; i < KM + 1; ++i) acc[i] = 0.0;
  for (int64_t base = wglob * RPW; base < a.n; base += wstride * RPW) {  // warp-uniform loop
    const int64_t r = base + grp;
    const bool valid = r < a.n;
    double t = 0.0;
    if (valid) {
      const int b = a.rp[r], e = a.rp[r + 1];
      for (int p = b + sub; p < e; p += CSR_G) t += a.va[p] * __ldg(a.xg + a.ci[p]);
    }
#pragma unroll
    for (int o = CSR_G / 2; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (valid && sub == 0) {
      if (a.mode == 1) {
        const double rr = a.f[r] - t;
        a.out[r] = rr;
        acc[0] += rr * rr;
      } else {
        a.out[r] = t;
        acc[0] += t * t;
#pragma unroll
        for (int l = 0; l < KM; ++l)
          if (l < a.nw) acc[1 + l] += a.W[(int64_t)(a.lo + l) * a.ld + r] * t;
      }
    }
  }
  __shared__ double R[KM + 1];
  block_sum_n<KM + 1>(acc, red, R);
  if (tid == 0) {
    for (int i = 0; i < SKS_NP; ++i)
      a.partials[(int64_t)blockIdx.x * SKS_NP + i] = (i < KM + 1) ? R[i] : 0.0;
  }
}

// Row-block SpMV (SKS_CSR_V2=1; measured SLOWER than csr_spmv_kernel at C4 -- 433-500 vs 254 us per launch,
// ncu: mio_throttle 57 / lg_throttle 16 warps per issue, issue active 5%: the burst of independent 32-address
// x gathers per thread saturates the memory-instruction queues; profiles/r02/csr_ab_r02.txt): a CTA takes 256
// consecutive rows; its
// threads walk the rows' contiguous nonzero range [rp[r0], rp[r0+256]) with a 256-entry stride (coalesced val /
// col_idx loads, several independent x gathers in flight per thread), stage the products in shared memory, then
// thread t sums row r0 + t (stride-17-style reads, conflict-free for odd row lengths).  Rows of a block whose nnz
// exceed the staging buffer are summed directly by their thread.  Same outputs and partial slots as
// csr_spmv_kernel (mode 0: mr and ||mr||^2, <w_i, mr>; mode 1: r = f - A x and ||r||^2).
constexpr int CSR2_R = 256;
constexpr int CSR2_CAP = 256 * 20;  // staged products per block (C4: 17 nnz per row -> 4352)
template <int KM>
__global__ void __launch_bounds__(CSR2_R) csr_spmv2_kernel(CsrArgs a) {
  __shared__ double red[SKS_NP * 32];
  __shared__ double prod[CSR2_CAP];
  const int tid = threadIdx.x;
  if (a.ctrl && (a.ctrl->exit_cols != 0 || a.ctrl->stop_col < 0x7fffffff)) return;
  double acc[KM + 1];
#pragma unroll
  for (int i = 0; i < KM + 1; ++i) acc[i] = 0.0;
  for (int64_t r0 = (int64_t)blockIdx.x * CSR2_R; r0 < a.n; r0 += (int64_t)gridDim.x * CSR2_R) {
    const int nr = (int)((a.n - r0) < CSR2_R ? (a.n - r0) : CSR2_R);
    const int b = a.rp[r0], e = a.rp[r0 + nr];
    const bool staged = (e - b) <= CSR2_CAP;
    if (staged) {  // all of this thread's column indices and values in flight, then all of its x gathers
      constexpr int NPT = CSR2_CAP / CSR2_R;
      int cix[NPT];
      double vv[NPT];
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        const int p = b + tid + i * CSR2_R;
        cix[i] = (p < e) ? __ldg(a.ci + p) : 0;
        vv[i] = (p < e) ? __ldg(a.va + p) : 0.0;
      }
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        const int p = b + tid + i * CSR2_R;
        if (p < e) prod[p - b] = vv[i] * __ldg(a.xg + cix[i]);
      }
    }
    __syncthreads();
    const int64_t r = r0 + tid;
    if (tid < nr) {
      const int rb = a.rp[r], re = a.rp[r + 1];
      double t = 0.0;
      if (staged) {
        for (int p = rb - b; p < re - b; ++p) t += prod[p];
      } else {
        for (int p = rb; p < re; ++p) t += a.va[p] * __ldg(a.xg + a.ci[p]);
      }
      if (a.mode == 1) {
        const double rr = a.f[r] - t;
        a.out[r] = rr;
        acc[0] += rr * rr;
      } else {
        a.out[r] = t;
        acc[0] += t * t;
#pragma unroll
        for (int l = 0; l < KM; ++l)
          if (l < a.nw) acc[1 + l] += a.W[(int64_t)(a.lo + l) * a.ld + r] * t;
      }
    }
    __syncthreads();  // prod is reused by the next block of rows
  }
  __shared__ double R[KM + 1];
  block_sum_n<KM + 1>(acc, red, R);
  if (tid == 0) {
    for (int i = 0; i < SKS_NP; ++i)
      a.partials[(int64_t)blockIdx.x * SKS_NP + i] = (i < KM + 1) ? R[i] : 0.0;
  }
}

struct OrthArgs {
  int64_t n;
  int j, k;
  double* W;
  int64_t ld;
  const double* mr;
  const double* pnorm;  // [grid_n][SKS_NP]: [0] = ||w_{j-1}||^2
  int grid_n;
  const double* pdot;   // [grid_s][SKS_NP]: [0] = ||mr||^2, [1+l] = <w_{lo+l}, mr>
  int grid_s;
  double* partials;     // out: [grid][SKS_NP], [0] = ||w_j||^2
  double* sigma;
  double* H;
  int ldH;
  double* mnorm;
  CtrlBlock* ctrl;
};

template <int KM>
__global__ void __launch_bounds__(256) csr_orth_kernel(OrthArgs a) {
  __shared__ double red[SKS_NP * 32];
  __shared__ double P[SKS_NP];
  __shared__ double Nn;
  __shared__ double cw[SKS_KMAX];
  __shared__ double cs;
  __shared__ int ok;
  const int tid = threadIdx.x;
  {
    double p[SKS_NP];
#pragma unroll
    for (int i = 0; i < SKS_NP; ++i) p[i] = 0.0;
    for (int b = tid; b < a.grid_s; b += blockDim.x)
#pragma unroll
      for (int i = 0; i < SKS_NP; ++i) p[i] += a.pdot[(int64_t)b * SKS_NP + i];
    block_sum_n<SKS_NP>(p, red, P);
    double q[1] = {0.0};
    for (int b = tid; b < a.grid_n; b += blockDim.x) q[0] += a.pnorm[(int64_t)b * SKS_NP];
    double o[1];
    block_sum_n<1>(q, red, o);
    if (tid == 0) Nn = o[0];
  }
  __syncthreads();
  const int j = a.j, jm = j - 1, lo = max(0, j - a.k);
  if (tid == 0) {
    ok = 1;
    if (a.ctrl->stop_col <= jm || a.ctrl->exit_cols != 0) ok = 0;
    const double N = Nn, nu = sqrt(N);
    bool bd = !(N > 0.0) || !isfinite(N);
    if (jm >= 1 && nu <= 1e-14 * a.mnorm[jm - 1]) bd = true;
    if (ok && bd) {
      ok = 0;
      if (blockIdx.x == 0) {
        a.ctrl->stop_col = jm;
        a.ctrl->breakdown = 1;
        if (jm >= 1) a.H[jm + (int64_t)(jm - 1) * a.ldH] = nu;
        if (jm == 0) a.ctrl->rnorm = nu;
      }
    }
    if (ok) {
      const double sg = 1.0 / nu;
      cs = sg;
      for (int i = lo; i <= jm; ++i) {
        const double si = (i == jm) ? sg : a.sigma[i];
        const double hi = sg * si * P[1 + i - lo];
        cw[i - lo] = -hi * si;
        if (blockIdx.x == 0) a.H[i + (int64_t)jm * a.ldH] = hi;
      }
      if (blockIdx.x == 0) {
        a.sigma[jm] = sg;
        a.mnorm[jm] = sg * sqrt(P[0]);
        if (jm >= 1) a.H[jm + (int64_t)(jm - 1) * a.ldH] = nu;
        if (jm == 0) a.ctrl->rnorm = nu;
      }
    }
  }
  __syncthreads();
  if (!ok) return;
  const int nw = jm - lo + 1;
  const double sg = cs;
  double* wj = a.W + (int64_t)j * a.ld;
  double acc[1] = {0.0};
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + tid; r < a.n; r += (int64_t)gridDim.x * blockDim.x) {
    double w = sg * a.mr[r];
#pragma unroll
    for (int l = 0; l < KM; ++l)
      if (l < nw) w += cw[l] * a.W[(int64_t)(lo + l) * a.ld + r];
    wj[r] = w;
    acc[0] += w * w;
  }
  double o[1];
  block_sum_n<1>(acc, red, o);
  if (tid == 0) {
    a.partials[(int64_t)blockIdx.x * SKS_NP] = o[0];
    for (int i = 1; i < SKS_NP; ++i) a.partials[(int64_t)blockIdx.x * SKS_NP + i] = 0.0;
  }
}

// start vector w_0 = v0 (copy) with ||w_0||^2 partials
__global__ void copy_norm_kernel(int64_t n, const double* __restrict__ src, double* __restrict__ dst,
                                 double* __restrict__ partials) {
  __shared__ double red[32];
  double acc[1] = {0.0};
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const double v = src[r];
    dst[r] = v;
    acc[0] += v * v;
  }
  double o[1];
  block_sum_n<1>(acc, red, o);
  if (threadIdx.x == 0) {
    partials[(int64_t)blockIdx.x * SKS_NP] = o[0];
    for (int i = 1; i < SKS_NP; ++i) partials[(int64_t)blockIdx.x * SKS_NP + i] = 0.0;
  }
}

// ------------------------------------------------------------------------------
static int csr_km(int k) { return k <= 2 ? 2 : (k <= 4 ? 4 : 8); }

#ifndef CSR_ELL_CH
#define CSR_ELL_CH 6  // entries (x gathers) in flight per thread (C4 sweep: 2 181, 3 183, 4 152, 6 147, 8 184, 16 157, 17 154 us)
#endif
// ELL SpMV (one thread per row, column-major [w][n] arrays: the k-th entries of 32 consecutive rows are one
// coalesced load, and each thread has 8 independent x gathers in flight).  Same outputs and partial slots as
// csr_spmv_kernel; row sums in entry order.
#ifndef CSR_ELL_T
#define CSR_ELL_T 256  // threads per CTA (the grid is the partial-slot count, 4 x SMs)
#endif
template <int KM>
__global__ void __launch_bounds__(CSR_ELL_T) csr_ell_kernel(CsrArgs a, const int32_t* __restrict__ eci,
                                                       const double* __restrict__ eva, int w) {
  __shared__ double red[SKS_NP * 32];
  const int tid = threadIdx.x;
  if (a.ctrl && (a.ctrl->exit_cols != 0 || a.ctrl->stop_col < 0x7fffffff)) return;
  double acc[KM + 1];
#pragma unroll
  for (int i = 0; i < KM + 1; ++i) acc[i] = 0.0;
  const int64_t n = a.n;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + tid; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    double t = 0.0;
    int k = 0;
    for (; k + CSR_ELL_CH <= w; k += CSR_ELL_CH) {
      int c[CSR_ELL_CH];
      double v[CSR_ELL_CH], x[CSR_ELL_CH];
#pragma unroll
      for (int u = 0; u < CSR_ELL_CH; ++u) {
        c[u] = __ldcs(eci + (int64_t)(k + u) * n + r);
        v[u] = __ldcs(eva + (int64_t)(k + u) * n + r);
      }
#pragma unroll
      for (int u = 0; u < CSR_ELL_CH; ++u) x[u] = __ldg(a.xg + c[u]);
#pragma unroll
      for (int u = 0; u < CSR_ELL_CH; ++u) t += v[u] * x[u];
    }
    for (; k < w; ++k) t += __ldcs(eva + (int64_t)k * n + r) * __ldg(a.xg + __ldcs(eci + (int64_t)k * n + r));
    if (a.mode == 1) {
      const double rr = a.f[r] - t;
      a.out[r] = rr;
      acc[0] += rr * rr;
    } else {
      a.out[r] = t;
      acc[0] += t * t;
#pragma unroll
      for (int l = 0; l < KM; ++l)
        if (l < a.nw) acc[1 + l] += a.W[(int64_t)(a.lo + l) * a.ld + r] * t;
    }
  }
  __shared__ double R[KM + 1];
  block_sum_n<KM + 1>(acc, red, R);
  if (tid == 0) {
    for (int i = 0; i < SKS_NP; ++i)
      a.partials[(int64_t)blockIdx.x * SKS_NP + i] = (i < KM + 1) ? R[i] : 0.0;
  }
}

__global__ void csr_max_row_kernel(int64_t n, const int32_t* __restrict__ rp, int* out) {
  int m = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x)
    m = max(m, rp[r + 1] - rp[r]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

__global__ void csr_to_ell_kernel(int64_t n, const int32_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                  const double* __restrict__ va, int w, int32_t* __restrict__ eci,
                                  double* __restrict__ eva) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int b = rp[r], len = rp[r + 1] - b;
    for (int k = 0; k < w; ++k) {
      eci[(int64_t)k * n + r] = k < len ? ci[b + k] : 0;
      eva[(int64_t)k * n + r] = k < len ? va[b + k] : 0.0;
    }
  }
}

cudaError_t launch_csr_max_row(int64_t n, const int32_t* rp, int* out, cudaStream_t st) {
  cudaMemsetAsync(out, 0, sizeof(int), st);
  csr_max_row_kernel<<<592, 256, 0, st>>>(n, rp, out);
  return cudaGetLastError();
}

cudaError_t launch_csr_to_ell(int64_t n, const int32_t* rp, const int32_t* ci, const double* va, int w, int32_t* eci,
                              double* eva, cudaStream_t st) {
  csr_to_ell_kernel<<<592, 256, 0, st>>>(n, rp, ci, va, w, eci, eva);
  return cudaGetLastError();
}

cudaError_t launch_csr_spmv(int64_t n, const int32_t* rp, const int32_t* ci, const double* va, const double* xg,
                            double* out, const double* f, int mode, const double* W, int64_t ld, int lo, int nw,
                            int k, double* partials, int grid, cudaStream_t st, const CtrlBlock* ctrl,
                            const int32_t* ell_ci, const double* ell_va, int ell_w) {
  CsrArgs a{n, rp, ci, va, xg, out, f, mode, W, ld, lo, nw, partials, ctrl};
  if (ell_w > 0) {
    switch (csr_km(k)) {
      case 2: csr_ell_kernel<2><<<grid, CSR_ELL_T, 0, st>>>(a, ell_ci, ell_va, ell_w); break;
      case 4: csr_ell_kernel<4><<<grid, CSR_ELL_T, 0, st>>>(a, ell_ci, ell_va, ell_w); break;
      default: csr_ell_kernel<8><<<grid, CSR_ELL_T, 0, st>>>(a, ell_ci, ell_va, ell_w); break;
    }
    return cudaGetLastError();
  }
  static int v1 = -1;
  if (v1 < 0) {
    const char* e = getenv("SKS_CSR_V2");
    v1 = (e && e[0] == '1') ? 0 : 1;
  }
  if (v1) {
    switch (csr_km(k)) {
      case 2: csr_spmv_kernel<2><<<grid, 256, 0, st>>>(a); break;
      case 4: csr_spmv_kernel<4><<<grid, 256, 0, st>>>(a); break;
      default: csr_spmv_kernel<8><<<grid, 256, 0, st>>>(a); break;
    }
    return cudaGetLastError();
  }
  switch (csr_km(k)) {
    case 2: csr_spmv2_kernel<2><<<grid, CSR2_R, 0, st>>>(a); break;
    case 4: csr_spmv2_kernel<4><<<grid, CSR2_R, 0, st>>>(a); break;
    default: csr_spmv2_kernel<8><<<grid, CSR2_R, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_csr_orth(int64_t n, int j, int k, double* W, int64_t ld, const double* mr, const double* pnorm,
                            int grid_n, const double* pdot, int grid_s, double* partials, double* sigma, double* H,
                            int ldH, double* mnorm, CtrlBlock* ctrl, int grid, cudaStream_t st) {
  OrthArgs a{n, j, k, W, ld, mr, pnorm, grid_n, pdot, grid_s, partials, sigma, H, ldH, mnorm, ctrl};
  switch (csr_km(k)) {
    case 2: csr_orth_kernel<2><<<grid, 256, 0, st>>>(a); break;
    case 4: csr_orth_kernel<4><<<grid, 256, 0, st>>>(a); break;
    default: csr_orth_kernel<8><<<grid, 256, 0, st>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_copy_norm(int64_t n, const double* src, double* dst, double* partials, int grid,
                             cudaStream_t st) {
  copy_norm_kernel<<<grid, 256, 0, st>>>(n, src, dst, partials);
  return cudaGetLastError();
}

}  // namespace sks
