// svd.cu -- the small side of stabilised sRR (Sec. "Stabilization"; reading O33).
//
// When the sketched basis is numerically rank-deficient (kappa_2(SB) >~ 1/u), sRR is
// regularised by a truncated SVD  SB = U Sigma V^* + E  and the pencil (U^* SAB V) z = theta Sigma z.
// Two kernels:
//
//   * jacobi_svd_kernel: one-sided (Hestenes) Jacobi SVD of SB (s x d) in one CTA -- column pairs
//     rotated until mutually orthogonal (|a_p . a_q| <= sqrt(s) u ||a_p|| ||a_q||, the dgesvj
//     criterion; columns below u ||SB||_F are numerically zero and left alone), round-robin (circle-method) pair
//     order so that the pairs of a round are disjoint and processed by different warps, fixed
//     reduction order (bitwise reproducible).  Sigma = column norms, sorted descending; Ut = columns
//     / sigma; the rank r = #{sigma_i >= sigma_1 / tol}.  One-sided Jacobi computes the small singular
//     values to high relative accuracy, which the truncation decision needs (the Gram matrix SB^T SB
//     would square kappa).
//   * hess_reduce_kernel: Householder reduction of M_r to Hessenberg form (the Francis QR and the
//     inverse iteration take Hessenberg input), the reflectors accumulated into V_r;
//   * small_gemm_kernel: C = diag(rs) op(A) op(B) in FP64 (16 x 16 tiles through shared memory) for
//     U_r^T SAB, M_r = Sigma_r^-1 (U_r^T SAB) V_r and y = (V_r Q) z.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace sks {

constexpr int SV_THREADS = 1024;
constexpr int SV_WARPS = SV_THREADS / 32;

__device__ __forceinline__ double sv_warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Mi: rows x n (column-major, ld ldm).  work: rows n + n^2 doubles (A, Vw).  Outputs: sigma[n]
// descending, Ut (rows x n, ld rows: left singular vectors), Vs (n x n, ld n), out[0] = rank r,
// out[1] = sweeps, out[2] = 1 if converged.
__global__ void __launch_bounds__(SV_THREADS, 1)
    jacobi_svd_kernel(const double* __restrict__ Mi, int ldm, int rows, int n, double tol, int max_sweeps,
                      double* __restrict__ work, double* __restrict__ sigma, double* __restrict__ Ut,
                      double* __restrict__ Vs, int* __restrict__ out) {
  double* A = work;
  double* Vw = work + (size_t)rows * n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  __shared__ int rotated;
  __shared__ double fro[SV_WARPS];
  double f2 = 0.0;
  for (int64_t e = tid; e < (int64_t)rows * n; e += SV_THREADS) {
    const int i = (int)(e % rows), j = (int)(e / rows);
    const double v = Mi[i + (int64_t)j * ldm];
    A[e] = v;
    f2 = fma(v, v, f2);
  }
  for (int64_t e = tid; e < (int64_t)n * n; e += SV_THREADS) Vw[e] = (e % n == e / n) ? 1.0 : 0.0;
  f2 = sv_warp_sum(f2);
  if (lane == 0) fro[wid] = f2;
  __syncthreads();
  double F2 = 0.0;
  for (int w = 0; w < SV_WARPS; ++w) F2 += fro[w];
  const double tiny = 1.2e-32 * F2;                     // (u ||SB||_F)^2: a numerically zero column
  const double ctol = sqrt((double)rows) * 2.220446049250313e-16;
  const int N = n + (n & 1);  // circle method on an even number of players (index n = bye)
  int sweep = 0, conv = 0;
  for (; sweep < max_sweeps; ++sweep) {
    if (tid == 0) rotated = 0;
    __syncthreads();
    for (int round = 0; round < N - 1; ++round) {
      for (int i = wid; i < N / 2; i += SV_WARPS) {
        int p, q;
        if (i == 0) {
          p = N - 1;
          q = round;
        } else {
          p = (round + i) % (N - 1);
          q = (round - i + N - 1) % (N - 1);
        }
        if (p >= n || q >= n) continue;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double* ap = A + (int64_t)p * rows;
        double* aq = A + (int64_t)q * rows;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < rows; r += 32) {
          const double x = ap[r], y = aq[r];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = sv_warp_sum(al);
        be = sv_warp_sum(be);
        ga = sv_warp_sum(ga);
        if (ga == 0.0 || al <= tiny || be <= tiny || fabs(ga) <= ctol * sqrt(al) * sqrt(be)) continue;
        // Hestenes rotation: zeroes a_p . a_q (Golub-Van Loan Alg. 8.5.2 on the 2x2 Gram block)
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
        for (int r = lane; r < rows; r += 32) {
          const double x = ap[r], y = aq[r];
          ap[r] = cs * x - sn * y;
          aq[r] = sn * x + cs * y;
        }
        double* vp = Vw + (int64_t)p * n;
        double* vq = Vw + (int64_t)q * n;
        for (int r = lane; r < n; r += 32) {
          const double x = vp[r], y = vq[r];
          vp[r] = cs * x - sn * y;
          vq[r] = sn * x + cs * y;
        }
        if (lane == 0) rotated = 1;  // benign race: every writer stores 1
      }
      __syncthreads();
    }
    const int any = rotated;
    __syncthreads();
    if (!any) {
      conv = 1;
      ++sweep;
      break;
    }
  }
  // ---- singular values = column norms; sort descending (ties: lower index first)
  for (int j = wid; j < n; j += SV_WARPS) {
    double s2 = 0.0;
    for (int r = lane; r < rows; r += 32) s2 = fma(A[(int64_t)j * rows + r], A[(int64_t)j * rows + r], s2);
    s2 = sv_warp_sum(s2);
    if (lane == 0) sigma[j] = sqrt(s2);  // unsorted for now
  }
  __syncthreads();
  extern __shared__ double sv_sm[];  // [n] sorted sigma, [n] int rank
  int* rk = reinterpret_cast<int*>(sv_sm + n);
  for (int j = tid; j < n; j += SV_THREADS) {
    const double sj = sigma[j];
    int r = 0;
    for (int k = 0; k < n; ++k) {
      const double sk = sigma[k];
      r += (sk > sj) || (sk == sj && k < j);
    }
    rk[j] = r;
    sv_sm[r] = sj;
  }
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)rows * n; e += SV_THREADS) {
    const int r = (int)(e % rows), j = (int)(e / rows);
    const int dst = rk[j];
    const double sj = sv_sm[dst];
    Ut[(int64_t)dst * rows + r] = sj > 0.0 ? A[e] / sj : 0.0;
  }
  for (int64_t e = tid; e < (int64_t)n * n; e += SV_THREADS) {
    const int r = (int)(e % n), j = (int)(e / n);
    Vs[(int64_t)rk[j] * n + r] = Vw[e];
  }
  __syncthreads();
  for (int j = tid; j < n; j += SV_THREADS) sigma[j] = sv_sm[j];
  if (tid == 0) {
    const double s0 = sv_sm[0];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (sv_sm[j] > 0.0 && sv_sm[j] * tol >= s0);
    out[0] = r;
    out[1] = sweep;
    out[2] = conv;
  }
}

// ---- multi-CTA version (rows, n <= 32 * JR_RPL): the pairs of a round are spread over every warp of a
// cooperative grid (one grid barrier per round); each warp holds its two columns in registers for
// the dots and the rotation (one pass over A per pair).  Same pair order, reductions and criterion
// and per-pair arithmetic as jacobi_svd_kernel.
constexpr int JR_RPL = 24;         // rows per lane held in registers (rows <= 768)
#ifndef JC_THREADS_DEF
#define JC_THREADS_DEF 64
#endif
constexpr int JC_THREADS = JC_THREADS_DEF;  // warps per CTA x 32
constexpr int JC_WARPS = JC_THREADS / 32;

__device__ __forceinline__ void jc_grid_barrier(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      atomicAdd(const_cast<unsigned*>(gen), 1u);
    } else {
      while (*gen == g) __nanosleep(64);
    }
    __threadfence();
  }
  __syncthreads();
}

// sync[0] = count, sync[1] = generation, sync[2..3] = per-sweep-parity rotation flags, sync[4] = F2 bits;
// all zero at launch.
__global__ void __launch_bounds__(JC_THREADS)
    jacobi_svd_coop_kernel(const double* __restrict__ Mi, int ldm, int rows, int n, int max_sweeps,
                           double* __restrict__ work, unsigned* __restrict__ sync, double* __restrict__ f2part,
                           int* __restrict__ out) {
  double* A = work;
  double* Vw = work + (size_t)rows * n;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int gw = blockIdx.x * JC_WARPS + wid, nw = gridDim.x * JC_WARPS;
  const unsigned nb = gridDim.x;
  // ---- copy, V = I, ||M||_F^2 in a fixed order (per-warp partials, summed by every thread)
  const int64_t gt = (int64_t)blockIdx.x * JC_THREADS + threadIdx.x;
  const int64_t nthr = (int64_t)nb * JC_THREADS;
  for (int64_t e = gt; e < (int64_t)n * n; e += nthr) Vw[e] = (e % n == e / n) ? 1.0 : 0.0;
  for (int c = gw; c < n; c += nw) {  // warp per column: fixed reduction order per column
    double f2 = 0.0;
    for (int r = lane; r < rows; r += 32) {
      const double v = Mi[r + (int64_t)c * ldm];
      A[r + (int64_t)c * rows] = v;
      f2 = fma(v, v, f2);
    }
    f2 = sv_warp_sum(f2);
    if (lane == 0) f2part[c] = f2;
  }
  jc_grid_barrier(sync, sync + 1, nb);
  double F2 = 0.0;
  for (int c = 0; c < n; ++c) F2 += f2part[c];
  const double tiny = 1.2e-32 * F2;
  const double ctol = sqrt((double)rows) * 2.220446049250313e-16;
  const int N = n + (n & 1);
  int sweep = 0, conv = 0;
  for (; sweep < max_sweeps; ++sweep) {
    for (int round = 0; round < N - 1; ++round) {
      for (int i = gw; i < N / 2; i += nw) {
        int p, q;
        if (i == 0) {
          p = N - 1;
          q = round;
        } else {
          p = (round + i) % (N - 1);
          q = (round - i + N - 1) % (N - 1);
        }
        if (p >= n || q >= n) continue;
        if (p > q) {
          const int t = p;
          p = q;
          q = t;
        }
        double* ap = A + (int64_t)p * rows;
        double* aq = A + (int64_t)q * rows;
        double x[JR_RPL], y[JR_RPL];
#pragma unroll
        for (int u = 0; u < JR_RPL; ++u) {
          const int r = lane + 32 * u;
          x[u] = r < rows ? ap[r] : 0.0;
          y[u] = r < rows ? aq[r] : 0.0;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
#pragma unroll
        for (int u = 0; u < JR_RPL; ++u) {
          al = fma(x[u], x[u], al);
          be = fma(y[u], y[u], be);
          ga = fma(x[u], y[u], ga);
        }
        al = sv_warp_sum(al);
        be = sv_warp_sum(be);
        ga = sv_warp_sum(ga);
        if (ga == 0.0 || al <= tiny || be <= tiny || fabs(ga) <= ctol * sqrt(al) * sqrt(be)) continue;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
#pragma unroll
        for (int u = 0; u < JR_RPL; ++u) {
          const int r = lane + 32 * u;
          if (r < rows) {
            ap[r] = cs * x[u] - sn * y[u];
            aq[r] = sn * x[u] + cs * y[u];
          }
        }
        double* vp = Vw + (int64_t)p * n;
        double* vq = Vw + (int64_t)q * n;
#pragma unroll
        for (int u = 0; u < JR_RPL; ++u) {  // all loads in flight before the stores
          const int r = lane + 32 * u;
          x[u] = r < n ? vp[r] : 0.0;
          y[u] = r < n ? vq[r] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < JR_RPL; ++u) {
          const int r = lane + 32 * u;
          if (r < n) {
            vp[r] = cs * x[u] - sn * y[u];
            vq[r] = sn * x[u] + cs * y[u];
          }
        }
        if (lane == 0) atomicOr(sync + 2 + (sweep & 1), 1u);
      }
      jc_grid_barrier(sync, sync + 1, nb);
      // the next sweep's flag was last read at the end of the previous sweep; every block has passed
      // that read once it has passed this round's barrier
      if (round == 0 && blockIdx.x == 0 && threadIdx.x == 0) sync[2 + ((sweep + 1) & 1)] = 0u;
    }
    const unsigned any = *((volatile unsigned*)(sync + 2 + (sweep & 1)));
    if (!any) {
      conv = 1;
      ++sweep;
      break;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    out[1] = sweep;
    out[2] = conv;
  }
}

// finishing pass of the multi-CTA version (one CTA): norms, sort, U, V, rank
__global__ void __launch_bounds__(SV_THREADS, 1)
    jacobi_svd_finish_kernel(int rows, int n, double tol, const double* __restrict__ work,
                             double* __restrict__ sigma, double* __restrict__ Ut, double* __restrict__ Vs,
                             int* __restrict__ out) {
  const double* A = work;
  const double* Vw = work + (size_t)rows * n;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int j = wid; j < n; j += SV_WARPS) {
    double s2 = 0.0;
    for (int r = lane; r < rows; r += 32) s2 = fma(A[(int64_t)j * rows + r], A[(int64_t)j * rows + r], s2);
    s2 = sv_warp_sum(s2);
    if (lane == 0) sigma[j] = sqrt(s2);
  }
  __syncthreads();
  extern __shared__ double sv_sm2[];
  int* rk = reinterpret_cast<int*>(sv_sm2 + n);
  for (int j = tid; j < n; j += SV_THREADS) {
    const double sj = sigma[j];
    int r = 0;
    for (int k = 0; k < n; ++k) {
      const double sk = sigma[k];
      r += (sk > sj) || (sk == sj && k < j);
    }
    rk[j] = r;
    sv_sm2[r] = sj;
  }
  __syncthreads();
  for (int64_t e = tid; e < (int64_t)rows * n; e += SV_THREADS) {
    const int r = (int)(e % rows), j = (int)(e / rows);
    const int dst = rk[j];
    const double sj = sv_sm2[dst];
    Ut[(int64_t)dst * rows + r] = sj > 0.0 ? A[e] / sj : 0.0;
  }
  for (int64_t e = tid; e < (int64_t)n * n; e += SV_THREADS) {
    const int r = (int)(e % n), j = (int)(e / n);
    Vs[(int64_t)rk[j] * n + r] = Vw[e];
  }
  __syncthreads();
  for (int j = tid; j < n; j += SV_THREADS) sigma[j] = sv_sm2[j];
  if (tid == 0) {
    const double s0 = sv_sm2[0];
    int r = 0;
    for (int j = 0; j < n; ++j) r += (sv_sm2[j] > 0.0 && sv_sm2[j] * tol >= s0);
    out[0] = r;
  }
}

// work: rows n + n^2 doubles, plus (multi-CTA path) 8 unsigned + n doubles of scratch at its end.
cudaError_t launch_jacobi_svd(const double* M, int ldm, int rows, int n, double tol, int max_sweeps, double* work,
                              double* sigma, double* Ut, double* Vs, int* out, cudaStream_t st) {
  const size_t smem = sizeof(double) * n + sizeof(int) * n;
  static int force_single = -1;
  if (force_single < 0) force_single = getenv("SKS_SVD_SINGLE") ? 1 : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(jacobi_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(jacobi_svd_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (rows > 32 * JR_RPL || n > 32 * JR_RPL || force_single) {
    jacobi_svd_kernel<<<1, SV_THREADS, smem, st>>>(M, ldm, rows, n, tol, max_sweeps, work, sigma, Ut, Vs, out);
    return cudaGetLastError();
  }
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_svd_coop_kernel, JC_THREADS, 0);
  const int pairs = (n + 1) / 2;
  int grid = std::min((pairs + JC_WARPS - 1) / JC_WARPS, nsm * std::max(per_sm, 1));
  grid = std::max(grid, 1);
  double* scratch = work + (size_t)rows * n + (size_t)n * n;
  unsigned* sync = reinterpret_cast<unsigned*>(scratch);
  double* f2part = scratch + 8;
  cudaError_t e = cudaMemsetAsync(sync, 0, 8 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&M, (void*)&ldm, (void*)&rows, (void*)&n, (void*)&max_sweeps, (void*)&work, (void*)&sync,
                  (void*)&f2part, (void*)&out};
  e = cudaLaunchCooperativeKernel((const void*)jacobi_svd_coop_kernel, dim3(grid), dim3(JC_THREADS), args, 0, st);
  if (e != cudaSuccess) return e;
  jacobi_svd_finish_kernel<<<1, SV_THREADS, smem, st>>>(rows, n, tol, work, sigma, Ut, Vs, out);
  return cudaGetLastError();
}

// ---- Householder reduction of M (n x n, ld ldm) to upper Hessenberg form H = Q^T M Q, in place, with
// the reflectors also applied from the right to V (vrows x n, ld ldv): V <- V Q.  The eigen-solvers
// (hqr, the Hessenberg inverse iteration) need Hessenberg input; Mhat from the recurrence is Hessenberg
// by construction (O28), the stabilised M_r is not.  One CTA; reflector v_j in shared memory.
__global__ void __launch_bounds__(SV_THREADS, 1)
    hess_reduce_kernel(double* __restrict__ M, int n, int ldm, double* __restrict__ V, int vrows, int ldv) {
  extern __shared__ double hv[];  // [n] reflector
  __shared__ double red[SV_WARPS];
  __shared__ double sh_beta, sh_alpha;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  for (int j = 0; j + 2 < n; ++j) {
    const int m0 = j + 1, len = n - m0;  // reflector acts on rows/cols m0 .. n-1
    // ---- x = M[m0:, j]; v = x - alpha e_1, alpha = -sign(x_0) ||x||
    double ss = 0.0;
    for (int i = tid; i < len; i += SV_THREADS) {
      const double x = M[(m0 + i) + (int64_t)j * ldm];
      hv[i] = x;
      ss = fma(x, x, ss);
    }
    ss = sv_warp_sum(ss);
    if (lane == 0) red[wid] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < SV_WARPS; ++q) t += red[q];
      const double x0 = hv[0];
      const double tail = t - x0 * x0;
      if (tail <= 0.0) {  // already Hessenberg in this column
        sh_beta = 0.0;
      } else {
        const double nx = sqrt(t);
        const double alpha = x0 >= 0.0 ? -nx : nx;
        hv[0] = x0 - alpha;
        sh_alpha = alpha;
        sh_beta = 1.0 / (nx * (nx + fabs(x0)));  // 2 / (v^T v)
      }
    }
    __syncthreads();
    const double beta = sh_beta;
    if (beta == 0.0) continue;  // CTA-uniform
    // ---- left: M[m0:, j+1:] -= beta v (v^T M[m0:, j+1:]); column j becomes alpha e_1
    for (int c = j + 1 + wid; c < n; c += SV_WARPS) {
      double* col = M + (int64_t)c * ldm + m0;
      double t = 0.0;
      for (int i = lane; i < len; i += 32) t = fma(hv[i], col[i], t);
      t = sv_warp_sum(t) * beta;
      for (int i = lane; i < len; i += 32) col[i] = fma(-t, hv[i], col[i]);
    }
    for (int i = tid; i < len; i += SV_THREADS) M[(m0 + i) + (int64_t)j * ldm] = (i == 0) ? sh_alpha : 0.0;
    __syncthreads();
    // ---- right: M[:, m0:] -= beta (M[:, m0:] v) v^T ; V[:, m0:] likewise
    for (int r = tid; r < n + vrows; r += SV_THREADS) {
      double* base = r < n ? M + r : V + (r - n);
      const int64_t ld = r < n ? ldm : ldv;
      double t = 0.0;
      for (int i = 0; i < len; ++i) t = fma(base[(int64_t)(m0 + i) * ld], hv[i], t);
      t *= beta;
      for (int i = 0; i < len; ++i) base[(int64_t)(m0 + i) * ld] = fma(-t, hv[i], base[(int64_t)(m0 + i) * ld]);
    }
    __syncthreads();
  }
}

// ---- multi-CTA Householder reduction (same reflectors and update order per element as
// hess_reduce_kernel): every CTA forms the reflector of column j redundantly from global memory (no
// broadcast), the left update is spread over the grid's warps by column, the right update over its
// CTAs by 32-row blocks; two grid barriers per column.
constexpr int HC_THREADS = 256;
constexpr int HC_WARPS = HC_THREADS / 32;
__global__ void __launch_bounds__(HC_THREADS)
    hess_reduce_coop_kernel(double* __restrict__ M, int n, int ldm, double* __restrict__ V, int vrows, int ldv,
                            unsigned* __restrict__ sync) {
  extern __shared__ double hcv[];  // [n] reflector
  __shared__ double red[HC_WARPS];
  __shared__ double hpart[HC_WARPS * 32];
  __shared__ double sh_beta, sh_alpha;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int gw = blockIdx.x * HC_WARPS + wid, nwg = gridDim.x * HC_WARPS;
  const unsigned nb = gridDim.x;
  for (int j = 0; j + 2 < n; ++j) {
    const int m0 = j + 1, len = n - m0;
    double ss = 0.0;
    for (int i = tid; i < len; i += HC_THREADS) {
      const double x = M[(m0 + i) + (int64_t)j * ldm];
      hcv[i] = x;
      ss = fma(x, x, ss);
    }
    ss = sv_warp_sum(ss);
    if (lane == 0) red[wid] = ss;
    __syncthreads();
    if (tid == 0) {
      double t = 0.0;
      for (int q = 0; q < HC_WARPS; ++q) t += red[q];
      const double x0 = hcv[0];
      if (t - x0 * x0 <= 0.0) {
        sh_beta = 0.0;
      } else {
        const double nx = sqrt(t);
        const double alpha = x0 >= 0.0 ? -nx : nx;
        hcv[0] = x0 - alpha;
        sh_alpha = alpha;
        sh_beta = 1.0 / (nx * (nx + fabs(x0)));
      }
    }
    __syncthreads();
    const double beta = sh_beta;
    if (beta != 0.0) {  // grid-uniform (every CTA computed the same value)
      for (int c = j + 1 + gw; c < n; c += nwg) {
        double* col = M + (int64_t)c * ldm + m0;
        double t = 0.0;
        for (int i = lane; i < len; i += 32) t = fma(hcv[i], col[i], t);
        t = sv_warp_sum(t) * beta;
        for (int i = lane; i < len; i += 32) col[i] = fma(-t, hcv[i], col[i]);
      }
    }
    jc_grid_barrier(sync, sync + 1, nb);  // column j read by every CTA; left update done
    if (beta != 0.0) {
      if (blockIdx.x == 0)
        for (int i = tid; i < len; i += HC_THREADS) M[(m0 + i) + (int64_t)j * ldm] = (i == 0) ? sh_alpha : 0.0;
      // right update by 32-row blocks (lane = row, coalesced): the CTA's warps split the reflector
      // length into HC_WARPS chunks, partial sums combined in a fixed order in shared memory
      const int nrb = (n + vrows + 31) / 32;
      const int chunk = (len + HC_WARPS - 1) / HC_WARPS;
      const int i0 = wid * chunk, i1 = min(len, i0 + chunk);
      for (int rb = blockIdx.x; rb < nrb; rb += gridDim.x) {
        const int r = rb * 32 + lane;
        const bool ok = r < n + vrows;
        double* base = r < n ? M + r : V + (ok ? r - n : 0);
        const int64_t ld = r < n ? ldm : ldv;
        double t = 0.0;
        if (ok)
          for (int i = i0; i < i1; ++i) t = fma(base[(int64_t)(m0 + i) * ld], hcv[i], t);
        hpart[wid * 32 + lane] = t;
        __syncthreads();
        double tr = 0.0;
#pragma unroll
        for (int w = 0; w < HC_WARPS; ++w) tr += hpart[w * 32 + lane];
        tr *= beta;
        if (ok)
          for (int i = i0; i < i1; ++i) base[(int64_t)(m0 + i) * ld] = fma(-tr, hcv[i], base[(int64_t)(m0 + i) * ld]);
        __syncthreads();
      }
    }
    jc_grid_barrier(sync, sync + 1, nb);
  }
}

// scratch: 8 unsigned of device memory for the grid barrier (NULL: single-CTA kernel)
cudaError_t launch_hess_reduce(double* M, int n, int ldm, double* V, int vrows, int ldv, unsigned* scratch,
                               cudaStream_t st) {
  const size_t smem = sizeof(double) * n;
  static int force_single = -1;
  if (force_single < 0) force_single = getenv("SKS_HESS_SINGLE") ? 1 : 0;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(hess_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(hess_reduce_coop_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  if (scratch == nullptr || force_single) {
    hess_reduce_kernel<<<1, SV_THREADS, smem, st>>>(M, n, ldm, V, vrows, ldv);
    return cudaGetLastError();
  }
  int dev = 0, nsm = 0, per_sm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, hess_reduce_coop_kernel, HC_THREADS, smem);
  // a CTA per 32-row block of the right update, enough warps for the columns of the left update
  int grid = std::max((n + vrows + 31) / 32, (n + HC_WARPS - 1) / HC_WARPS);
  grid = std::max(1, std::min(grid, nsm * std::max(per_sm, 1)));
  cudaError_t e = cudaMemsetAsync(scratch, 0, 8 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {(void*)&M, (void*)&n, (void*)&ldm, (void*)&V, (void*)&vrows, (void*)&ldv, (void*)&scratch};
  e = cudaLaunchCooperativeKernel((const void*)hess_reduce_coop_kernel, dim3(grid), dim3(HC_THREADS), args, smem, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// C (M x N, ld ldc) = diag(rs) op(A) op(B); op(A) is M x K: A (ld lda) if !ta else A^T; op(B) is K x N.
// rs may be NULL (no row scaling); rs_inv != 0 scales row i by 1 / rs[i].
constexpr int SG = 16;
__global__ void __launch_bounds__(SG* SG)
    small_gemm_kernel(int M, int N, int K, const double* __restrict__ A, int lda, int ta,
                      const double* __restrict__ B, int ldb, int tb, const double* __restrict__ rs, int rs_inv,
                      double* __restrict__ Cm, int ldc) {
  __shared__ double As[SG][SG + 1], Bs[SG][SG + 1];
  const int tx = threadIdx.x % SG, ty = threadIdx.x / SG;
  const int i = blockIdx.y * SG + ty, j = blockIdx.x * SG + tx;
  double acc = 0.0;
  for (int k0 = 0; k0 < K; k0 += SG) {
    {  // As[ty][tx] = op(A)(blockIdx.y*SG + ty, k0 + tx)
      const int ai = blockIdx.y * SG + ty, ak = k0 + tx;
      As[ty][tx] = (ai < M && ak < K) ? (ta ? A[ak + (int64_t)ai * lda] : A[ai + (int64_t)ak * lda]) : 0.0;
    }
    {  // Bs[ty][tx] = op(B)(k0 + ty, blockIdx.x*SG + tx)
      const int bk = k0 + ty, bj = blockIdx.x * SG + tx;
      Bs[ty][tx] = (bk < K && bj < N) ? (tb ? B[bj + (int64_t)bk * ldb] : B[bk + (int64_t)bj * ldb]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SG; ++kk) acc = fma(As[ty][kk], Bs[kk][tx], acc);
    __syncthreads();
  }
  if (i < M && j < N) {
    double v = acc;
    if (rs) v = rs_inv ? v / rs[i] : v * rs[i];
    Cm[i + (int64_t)j * ldc] = v;
  }
}

cudaError_t launch_small_gemm(int M, int N, int K, const double* A, int lda, int ta, const double* B, int ldb,
                              int tb, const double* rs, int rs_inv, double* C, int ldc, cudaStream_t st) {
  if (M <= 0 || N <= 0) return cudaSuccess;
  dim3 grid((N + SG - 1) / SG, (M + SG - 1) / SG);
  small_gemm_kernel<<<grid, SG * SG, 0, st>>>(M, N, K, A, lda, ta, B, ldb, tb, rs, rs_inv, C, ldc);
  return cudaGetLastError();
}

}  // namespace sks
