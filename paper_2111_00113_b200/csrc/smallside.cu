// smallside.cu -- the s x d side of sGMRES / sRR on the device.
//
//  * form_cols:  sketched reduced-matrix columns from the basis sketch via the Arnoldi
//                recurrence  m_j = sum_i h_ij b_i + w_{j+1}, i.e.
//                S m_j = S w_{j+1} + sum_i h_ij sigma_i S w_i,
//                or plain  S b_j = sigma_j S w_j.
//  * incremental thin QR of the sketched matrix (Eq. sgmres-iterative-qr),
//    appended J columns at a time by block classical Gram-Schmidt with
//    re-orthogonalisation (BCGS2) against the explicit orthonormal U, then CGS2
//    inside the panel;  the residual s-vector  g - U_j U_j^T g  is updated column by
//    column so r_est,j (Eq. sgmres-iterative-soln, reading O14) is a plain norm
//    with no cancellation; early-exit test (reading O16).
//  * triangular solves (yhat = T^-1 U^T g), kappa(T) estimate,
//  * assembly x += B yhat (reading O13) and Ritz vectors X = B Y.
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sks {

// X[q*ldq + jj*ldj], columns jj = 0..J-1 correspond to basis index j = j0+jj.
// mode 0 (SAB):  X[:,jj] = gam_j SW[:, j+1] + sum_{i=max(0,j-k+1)}^{j} H[i,j] sigma_i SW[:, i]
// mode 1 (SB):   X[:,jj] = sigma_j SW[:, j]
// mode 2 (raw):  X[:,jj] = SW[:, j]
__global__ void form_cols_kernel(int mode, const double* __restrict__ SW, int s, int j0, int J, int k,
                                 const double* __restrict__ H, int ldH, const double* __restrict__ sigma,
                                 const double* __restrict__ gam, double* __restrict__ X, int64_t ldq, int64_t ldj) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= s * J) return;
  const int q = idx / J, jj = idx % J, j = j0 + jj;
  double v;
  if (mode == 1) {
    v = sigma[j] * SW[(int64_t)j * s + q];
  } else if (mode == 2) {
    v = SW[(int64_t)j * s + q];
  } else {
    v = gam[j] * SW[(int64_t)(j + 1) * s + q];
    const int lo = max(0, j - k + 1);
    for (int i = lo; i <= j; ++i) v += H[i + (int64_t)j * ldH] * sigma[i] * SW[(int64_t)i * s + q];
  }
  X[(int64_t)q * ldq + (int64_t)jj * ldj] = v;
}

// ------------------------------------------------------------------------------------
// Split-K fp64 GEMM for the two block Gram-Schmidt products of the sketched QR
// (BCGS2 projection of a panel X against the explicit U):
//   utx :  Z (j0 x J) = U[:, :j0]^T X          (A(m=i, k=q) = U[q + i*ldu]),  T[i, tc0+c] (+)= Z
//   xmuz:  X (s x J) -= U[:, :j0] Z            (A(m=q, k=i) = U[q + i*ldu])
// 32 x 32 output tiles, 32-deep k steps through shared memory, k split over gridDim.y CTAs;
// the last CTA of a tile (atomic ticket) adds the k-partials in ascending split order, so
// the result is bitwise reproducible.
// ------------------------------------------------------------------------------------
struct GemmArgs {
  const double* A;
  int64_t sAm, sAk;
  const double* B;  // K x J row-major (ld = J)
  int M, J, K, KC, KS;
  double* P;        // partials [KS][Mpad][32]
  int Mpad;
  int* cnt;         // one ticket per m tile (zero between calls)
  int mode;         // 0: utx, 1: xmuz
  double* Z;
  double* T;
  int ldT, tc0, tacc;
  double* X;
};

template <bool AK>
__global__ void __launch_bounds__(256) bgs_gemm_kernel(GemmArgs g) {
  __shared__ double As[32][33];
  __shared__ double Bs[32][33];
  __shared__ int last;
  const int tid = threadIdx.x, tx = tid & 31, ty = tid >> 5;
  const int m0 = blockIdx.x * 32, z = blockIdx.y;
  const int kb0 = z * g.KC, ke = min(g.K, kb0 + g.KC);
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int kb = kb0; kb < ke; kb += 32) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int e = tid + 256 * r;
      const int mm = AK ? (e >> 5) : (e & 31), kk = AK ? (e & 31) : (e >> 5);
      const int m = m0 + mm, k = kb + kk;
      As[kk][mm] = (m < g.M && k < ke) ? g.A[(int64_t)m * g.sAm + (int64_t)k * g.sAk] : 0.0;
      const int kk2 = e >> 5, nn = e & 31, k2 = kb + kk2;
      Bs[kk2][nn] = (k2 < ke && nn < g.J) ? g.B[(int64_t)k2 * g.J + nn] : 0.0;
    }
    __syncthreads();
#pragma unroll 8
    for (int kk = 0; kk < 32; ++kk) {
      const double b = Bs[kk][tx];
#pragma unroll
      for (int r = 0; r < 4; ++r) acc[r] += As[kk][ty * 4 + r] * b;
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) g.P[((int64_t)z * g.Mpad + m0 + ty * 4 + r) * 32 + tx] = acc[r];
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(&g.cnt[blockIdx.x], 1) == g.KS - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int m = m0 + ty * 4 + r;
    if (m >= g.M || tx >= g.J) continue;
    double v = 0.0;
    for (int zz = 0; zz < g.KS; ++zz) v += __ldcg(&g.P[((int64_t)zz * g.Mpad + m) * 32 + tx]);
    if (g.mode == 0) {
      g.Z[(int64_t)m * g.J + tx] = v;
      if (g.T) {
        double* t = g.T + m + (int64_t)(g.tc0 + tx) * g.ldT;
        *t = g.tacc ? (*t + v) : v;
      }
    } else {
      g.X[(int64_t)m * g.J + tx] -= v;
    }
  }
  if (tid == 0) g.cnt[blockIdx.x] = 0;
}

static cudaError_t launch_bgs_gemm(GemmArgs g, bool ak, double* ws, int* cnt, cudaStream_t st) {
  const int mt = (g.M + 31) / 32;
  int ks = (120 + mt - 1) / mt;
  ks = std::max(1, std::min(ks, 8));
  int kc = ((g.K + ks - 1) / ks + 31) / 32 * 32;
  ks = (g.K + kc - 1) / kc;
  g.KC = kc;
  g.KS = ks;
  g.Mpad = mt * 32;
  g.P = ws;
  g.cnt = cnt;
  dim3 grid(mt, ks);
  if (ak) bgs_gemm_kernel<true><<<grid, 256, 0, st>>>(g);
  else bgs_gemm_kernel<false><<<grid, 256, 0, st>>>(g);
  return cudaGetLastError();
}

size_t bgs_workspace_doubles(int s, int ncol) { return (size_t)8 * ((std::max(s, ncol) + 31) / 32 * 32) * 32; }

// One CTA: thin QR of the panel X (s x J row-major, already projected twice against U) by
// shifted Cholesky QR, three passes (sCholQR3: pass 1 factors X^T X + sigma I with
// sigma = 11 (sJ + J(J+1)) u ||X||_F^2, passes 2-3 are plain CholQR; orthogonality O(u) for
// kappa(X) up to O(1/u)).  Writes U[:, j0..j0+J), T[j0.., j0..] = R3 R2 R1, updates the
// residual vector rvec (length s): rho[j] = u_j^T r_{j-1}, rest[j] = ||r_j|| with the
// explicit vectors r_j = r - sum_{i<=j} rho_i u_i (one warp per j: no cancellation), and the
// early-exit test (reading O16).  A pivot that is not positive marks the panel rank deficient
// at that column (columns from there on are not used).
constexpr int PJ = SKS_JB;  // max panel width
constexpr int PL = PJ + 1;  // smem row stride of the 32 x 32 factors

__global__ void __launch_bounds__(1024) panel_kernel(double* __restrict__ X, int s, int J, int j0,
                                                     double* __restrict__ U, int ldu, double* __restrict__ T,
                                                     int ldT, double* __restrict__ rvec, double* __restrict__ rho,
                                                     double* __restrict__ rest, CtrlBlock* ctrl, int track_res,
                                                     int max_cols) {
  extern __shared__ double sm[];
  const int L = J + 1;               // odd smem row stride
  double* sX = sm;                   // s x J, row stride L
  double* sr = sX + (size_t)s * L;   // s
  __shared__ double G[PJ * PL];      // Gram / Cholesky factor of the current pass
  __shared__ double Rt[PJ * PL];     // accumulated R (upper)
  __shared__ double Rn[PJ * PL];     // scratch for the product
  __shared__ double rh[PJ];
  __shared__ int nbad;               // first rank-deficient column (J if none)
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, wid = tid >> 5;
  const int Jv = max(0, min(J, max_cols - j0));
  for (int i = tid; i < s * J; i += nt) sX[(i / J) * L + (i % J)] = X[i];
  if (track_res)
    for (int i = tid; i < s; i += nt) sr[i] = rvec[i];
  {
    const int i = tid >> 5, j = tid & 31;
    Rt[i * PL + j] = (i == j) ? 1.0 : 0.0;
  }
  if (tid == 0) nbad = Jv;
  __syncthreads();
  for (int pass = 0; pass < 3; ++pass) {
    const int Jc = nbad;  // columns still factored
    // ---- Gram G = X^T X on the FP64 tensor cores: warp t < 16 owns the 8x8 tile (t/4, t%4),
    //      mma.m8n8k4 over k = rows of X (A = X^T: A[m][k] = X[k][m]; B = X); columns >= Jc read as 0
    if (wid < 16) {
      const int mt = wid >> 2, ntl = wid & 3, lr = lane >> 2, lc = lane & 3;
      const int mcol = 8 * mt + lr, ncol = 8 * ntl + lr;
      const bool mok = mcol < Jc, nok = ncol < Jc;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;  // two accumulator pairs (independent DMMA chains)
      int q = 0;
      for (; q + 7 < s; q += 8) {
        const double a0 = mok ? sX[(q + lc) * L + mcol] : 0.0, b0 = nok ? sX[(q + lc) * L + ncol] : 0.0;
        const double a1 = mok ? sX[(q + 4 + lc) * L + mcol] : 0.0, b1 = nok ? sX[(q + 4 + lc) * L + ncol] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d0), "+d"(d1) : "d"(a0), "d"(b0));
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(e0), "+d"(e1) : "d"(a1), "d"(b1));
      }
      for (; q < s; q += 4) {
        const bool kok = q + lc < s;
        const double a0 = (mok && kok) ? sX[(q + lc) * L + mcol] : 0.0;
        const double b0 = (nok && kok) ? sX[(q + lc) * L + ncol] : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                     : "+d"(d0), "+d"(d1) : "d"(a0), "d"(b0));
      }
      const int gi = 8 * mt + lr, gj = 8 * ntl + 2 * lc;
      G[gi * PL + gj] = d0 + e0;
      G[gi * PL + gj + 1] = d1 + e1;
    }
    __syncthreads();
    // ---- Cholesky G = R^T R (upper R in place), right-looking over the whole CTA: thread (i, j)
    //      owns G[i][j]; per step one scalar (sqrt), one row scaling, one rank-1 trailing update
    __shared__ double csh[2];
    if (tid == 0) {
      double shift = 0.0;
      if (pass == 0) {
        double tr = 0.0;
        for (int l = 0; l < Jc; ++l) tr += G[l * PL + l];
        shift = 11.0 * ((double)s * Jc + (double)Jc * (Jc + 1)) * 1.1102230246251565e-16 * tr;
      }
      csh[0] = shift;
    }
    __syncthreads();
    if (pass == 0 && tid < Jc) G[tid * PL + tid] += csh[0];
    {
      const int ci = tid >> 5, cj = tid & 31;
      int bad = Jc;
      for (int k = 0; k < Jc; ++k) {
        __syncthreads();
        if (tid == 0) {
          const double d = G[k * PL + k];
          const bool okd = (d > 0.0) && isfinite(d);
          const double rk = okd ? sqrt(d) : 1.0;
          G[k * PL + k] = rk;
          csh[0] = 1.0 / rk;
          csh[1] = okd ? 1.0 : 0.0;
        }
        __syncthreads();
        if (csh[1] == 0.0) {
          bad = k;
          break;
        }
        if (tid > k && tid < Jc) G[k * PL + tid] *= csh[0];
        __syncthreads();
        if (ci > k && ci <= cj && cj < Jc) G[ci * PL + cj] = fma(-G[k * PL + ci], G[k * PL + cj], G[ci * PL + cj]);
      }
      if (tid == 0) nbad = bad;
    }
    __syncthreads();
    const int Jn = nbad;
    // ---- X <- X R^-1 (thread per row, forward substitution over the columns)
    for (int q = tid; q < s; q += nt) {
      double* xr = sX + q * L;
      for (int j = 0; j < Jn; ++j) {
        double v0 = xr[j], v1 = 0.0;  // two chains
        int i = 0;
        for (; i + 1 < j; i += 2) {
          v0 = fma(-xr[i], G[i * PL + j], v0);
          v1 = fma(-xr[i + 1], G[(i + 1) * PL + j], v1);
        }
        if (i < j) v0 = fma(-xr[i], G[i * PL + j], v0);
        xr[j] = (v0 + v1) / G[j * PL + j];
      }
    }
    // ---- Rt <- R Rt (upper triangular product)
    {
      const int i = tid >> 5, j = tid & 31;
      double v = 0.0;
      if (i <= j && j < Jn)
        for (int l = i; l <= j; ++l) v += G[i * PL + l] * Rt[l * PL + j];
      Rn[i * PL + j] = v;
    }
    __syncthreads();
    {
      const int i = tid >> 5, j = tid & 31;
      if (j < Jn) Rt[i * PL + j] = Rn[i * PL + j];
    }
    __syncthreads();
  }
  const int Jg = nbad;  // good columns
  // ---- outputs: U columns, T block
  for (int i = tid; i < s * Jg; i += nt) {
    const int q = i % s, c = i / s;
    U[q + (int64_t)(j0 + c) * ldu] = sX[q * L + c];
  }
  {
    const int i = tid >> 5, j = tid & 31;
    if (j < Jg && i < Jv) T[(j0 + i) + (int64_t)(j0 + j) * ldT] = (i <= j) ? Rt[i * PL + j] : 0.0;
  }
  if (track_res && Jg > 0) {
    // rho_c = u_c . r  (warp c)
    if (wid < Jg) {
      double t = 0.0;
      for (int q = lane; q < s; q += 32) t += sX[q * L + wid] * sr[q];
      t = warp_sum(t);
      if (lane == 0) rh[wid] = t;
    }
    __syncthreads();
    // rest_c = || r - sum_{i<=c} rho_i u_i ||  (warp c, explicit residual vector)
    if (wid < Jg) {
      double e = 0.0;
      for (int q = lane; q < s; q += 32) {
        double v = sr[q];
        for (int i = 0; i <= wid; ++i) v -= rh[i] * sX[q * L + i];
        e += v * v;
        if (wid == Jg - 1) rvec[q] = v;
      }
      e = warp_sum(e);
      if (lane == 0) {
        rho[j0 + wid] = rh[wid];
        rest[j0 + wid] = sqrt(e);
        Rn[wid] = sqrt(e);
      }
    }
    __syncthreads();
    if (tid == 0) {
      for (int c = 0; c < Jg; ++c) {
        ctrl->r_est_last = Rn[c];
        if (ctrl->exit_cols == 0 && Rn[c] <= ctrl->thr) ctrl->exit_cols = j0 + c + 1;
      }
    }
  }
  if (tid == 0) {
    if (Jg > 0) ctrl->qr_cols = j0 + Jg;
    if (Jg < Jv) ctrl->rank_def = 1;
  }
}

// kappa_2(T[:n,:n]) = sigma_max / sigma_min of the upper-triangular factor, estimated by
// power iteration on T^T T and inverse iteration (T^T T)^-1 (reading O25).  One CTA of 1024
// threads: products are row- / column-parallel with coalesced column reads, the triangular
// solves are blocked (32 x 32 diagonal blocks solved by one warp from shared memory, the
// off-diagonal updates by the whole CTA).
constexpr int CN_T = 1024;

__device__ __forceinline__ double cta_norm(const double* v, int n, double* red) {
  double t = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) t += v[i] * v[i];
  return sqrt(block_sum(t, red));
}

// y := T^-1 y (upper, backward) or T^-T y (forward), in place on shared y
__device__ void cta_trsv(const double* __restrict__ T, int ldT, int n, double* y, bool trans, double* blk) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  const int nb = (n + 31) / 32;
  for (int bb = 0; bb < nb; ++bb) {
    const int b = trans ? bb : nb - 1 - bb;
    const int i0 = b * 32, bs = min(32, n - i0);
    // diagonal block into shared memory (blk[r*33 + c] = T[i0+r, i0+c])
    for (int e = tid; e < 32 * 32; e += blockDim.x) {
      const int r = e & 31, c = e >> 5;
      blk[r * 33 + c] = (r < bs && c < bs && r <= c) ? T[(i0 + r) + (int64_t)(i0 + c) * ldT] : 0.0;
    }
    __syncthreads();
    if (wid == 0) {
      double yl = lane < bs ? y[i0 + lane] : 0.0;
      if (!trans) {
        for (int c = bs - 1; c >= 0; --c) {
          const double yc = __shfl_sync(0xffffffffu, yl, c) / blk[c * 33 + c];
          if (lane == c) yl = yc;
          if (lane < c) yl -= blk[lane * 33 + c] * yc;
        }
      } else {
        for (int c = 0; c < bs; ++c) {
          const double yc = __shfl_sync(0xffffffffu, yl, c) / blk[c * 33 + c];
          if (lane == c) yl = yc;
          if (lane > c && lane < bs) yl -= blk[c * 33 + lane] * yc;
        }
      }
      if (lane < bs) y[i0 + lane] = yl;
    }
    __syncthreads();
    if (!trans) {
      // y[0:i0) -= T[0:i0, i0:i0+bs) y_b
      for (int i = tid; i < i0; i += blockDim.x) {
        double t = 0.0;
        for (int c = 0; c < bs; ++c) t += T[i + (int64_t)(i0 + c) * ldT] * y[i0 + c];
        y[i] -= t;
      }
    } else {
      // y[l] -= T[i0:i0+bs, l]^T y_b for l >= i0+bs: warp per column
      for (int l = i0 + bs + wid; l < n; l += nw) {
        double t = lane < bs ? T[(i0 + lane) + (int64_t)l * ldT] * y[i0 + lane] : 0.0;
        t = warp_sum(t);
        if (lane == 0) y[l] -= t;
      }
    }
    __syncthreads();
  }
}

// back substitution T[:n,:n] y = b (upper, column-major), then out[i] = y[i]*scale[i] (scale may be
// NULL); also writes y to yout if non-NULL.  Blocked, one CTA (yhat = T^-1 U^T g).
__global__ void __launch_bounds__(CN_T) trsv_upper_kernel(const double* __restrict__ T, int ldT, int n,
                                                          const double* __restrict__ b,
                                                          const double* __restrict__ scale,
                                                          double* __restrict__ yout, double* __restrict__ out) {
  extern __shared__ double y[];
  __shared__ double blk[32 * 33];
  for (int i = threadIdx.x; i < n; i += blockDim.x) y[i] = b[i];
  __syncthreads();
  cta_trsv(T, ldT, n, y, false, blk);
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    if (yout) yout[i] = y[i];
    if (out) out[i] = scale ? y[i] * scale[i] : y[i];
  }
}

__global__ void __launch_bounds__(CN_T) cond_kernel(const double* __restrict__ T, int ldT, int n, int iters,
                                                    CtrlBlock* ctrl, double* __restrict__ out) {
  extern __shared__ double sm[];
  double* v = sm;
  double* u = sm + n;
  __shared__ double blk[32 * 33];
  __shared__ double red[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  // largest singular value: v <- T^T T v
  for (int i = tid; i < n; i += blockDim.x) v[i] = 1.0 / sqrt((double)n) * (1.0 + 0.01 * (i % 7));
  __syncthreads();
  double smax = 0.0;
  for (int it = 0; it < iters; ++it) {
    const double nv = cta_norm(v, n, red);
    for (int i = tid; i < n; i += blockDim.x) v[i] /= nv;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {  // u = T v (row-parallel, coalesced columns)
      double t = 0.0;
      for (int l = i; l < n; ++l) t += T[i + (int64_t)l * ldT] * v[l];
      u[i] = t;
    }
    __syncthreads();
    for (int l = wid; l < n; l += nw) {  // v = T^T u (warp per column)
      double t = 0.0;
      for (int i = lane; i <= l; i += 32) t += T[i + (int64_t)l * ldT] * u[i];
      t = warp_sum(t);
      if (lane == 0) v[l] = t;
    }
    __syncthreads();
    smax = sqrt(cta_norm(v, n, red));
  }
  // smallest singular value: v <- T^-1 T^-T v
  for (int i = tid; i < n; i += blockDim.x) v[i] = 1.0 / sqrt((double)n) * (1.0 + 0.01 * (i % 5));
  __syncthreads();
  double smin_inv = 0.0;
  for (int it = 0; it < iters; ++it) {
    const double nv = cta_norm(v, n, red);
    for (int i = tid; i < n; i += blockDim.x) v[i] /= nv;
    __syncthreads();
    cta_trsv(T, ldT, n, v, true, blk);
    cta_trsv(T, ldT, n, v, false, blk);
    smin_inv = sqrt(cta_norm(v, n, red));
  }
  if (tid == 0) {
    const double c = smax * smin_inv;
    if (ctrl) ctrl->cond = c;
    if (out) *out = c;
  }
}

// x[off + p] += sum_{i<nc} coef[i] W[off + p + i*ld]   (p < n)
__global__ void assemble_kernel(double* __restrict__ x, const double* __restrict__ W, int64_t ld, int64_t off,
                                int64_t n, const double* __restrict__ coef, const int* __restrict__ ncp,
                                int nc_max) {
  extern __shared__ double cs[];
  const int nc = min(*ncp, nc_max);
  for (int i = threadIdx.x; i < nc; i += blockDim.x) cs[i] = coef[i];
  __syncthreads();
  const int64_t n2 = n / 2;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n2; p += (int64_t)gridDim.x * blockDim.x) {
    double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
    const double* w = W + off + 2 * p;
    int i = 0;
    for (; i + 1 < nc; i += 2) {
      const double2 u = *reinterpret_cast<const double2*>(w + (int64_t)i * ld);
      const double2 v = *reinterpret_cast<const double2*>(w + (int64_t)(i + 1) * ld);
      a0 += cs[i] * u.x;
      a1 += cs[i] * u.y;
      b0 += cs[i + 1] * v.x;
      b1 += cs[i + 1] * v.y;
    }
    if (i < nc) {
      const double2 u = *reinterpret_cast<const double2*>(w + (int64_t)i * ld);
      a0 += cs[i] * u.x;
      a1 += cs[i] * u.y;
    }
    x[off + 2 * p] += a0 + b0;
    x[off + 2 * p + 1] += a1 + b1;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    double a = 0.0;
    for (int i = 0; i < nc; ++i) a += cs[i] * W[off + n - 1 + (int64_t)i * ld];
    x[off + n - 1] += a;
  }
}

// X_re/X_im[:, v] = sum_{i<nc} W[:, i] * sigma_i * Y(i, v)  (Y complex, yr/yi column-major ld = ldy)
// ---- Ritz vectors x_v = B y_v = W diag(sigma) y_v (Alg. 2), compacted.
// A conjugate pair (theta, conj theta) has y_v' = conj(y_v), so X_v' = conj(X_v), and a real theta
// has a real y: only the distinct real columns Re y, Im y are multiplied with W (C5: 10 instead
// of 22), each written to up to two outputs with a sign.  ritz_coef_kernel builds the compact
// coefficient matrix C = diag(sigma) [y columns] (nc x RV_MAXC) and the destination table.
constexpr int RV_MAXC = 24;

__global__ void ritz_coef_kernel(const double* __restrict__ sigma, const double* __restrict__ yr,
                                 const double* __restrict__ yi, int ldy, int nc, const double* __restrict__ th_re,
                                 const double* __restrict__ th_im, const int* __restrict__ nsel, int nmax,
                                 double* __restrict__ coef, int* __restrict__ meta) {
  __shared__ int src[RV_MAXC];  // compact column -> (v << 1) | imag
  __shared__ int ncomp;
  if (threadIdx.x == 0) {
    int dst[2 * RV_MAXC];
    for (int t = 0; t < 2 * RV_MAXC; ++t) dst[t] = 0;
    int pr[32];  // v -> compact column of Re y_v, or -1; paired flag via -2
    const int ns = min(*nsel, nmax);
    int nco = 0;
    for (int v = 0; v < ns && v < 32; ++v) {
      pr[v] = -1;
      if (th_im[v] == 0.0) {
        if (nco < RV_MAXC) {
          src[nco] = v << 1;
          dst[2 * nco] = 2 * v + 1;  // +Xr_v   (out id + 1, signed)
          pr[v] = nco++;
        }
        continue;
      }
      int u = -1;
      for (int w = 0; w < v; ++w)
        if (pr[w] >= 0 && th_im[w] != 0.0 && fabs(th_re[w] - th_re[v]) <= 1e-12 * fabs(th_re[v]) &&
            fabs(th_im[w] + th_im[v]) <= 1e-12 * fabs(th_im[v])) {
          u = w;
          break;
        }
      if (u >= 0) {  // X_v = conj(X_u)
        const int cr = pr[u];
        dst[2 * cr + 1] = 2 * v + 1;           // +Xr_v from Re
        dst[2 * (cr + 1) + 1] = -(2 * v + 2);  // -Xi_v from Im
        pr[u] = -2;
        continue;
      }
      if (nco + 2 <= RV_MAXC) {
        src[nco] = v << 1;
        dst[2 * nco] = 2 * v + 1;
        src[nco + 1] = (v << 1) | 1;
        dst[2 * (nco + 1)] = 2 * v + 2;  // +Xi_v
        pr[v] = nco;
        nco += 2;
      }
    }
    ncomp = nco;
    meta[0] = nco;
    for (int t = 0; t < 2 * RV_MAXC; ++t) meta[1 + t] = dst[t];
  }
  __syncthreads();
  const int nco = ncomp;
  for (int idx = threadIdx.x; idx < nc * RV_MAXC; idx += blockDim.x) {
    const int i = idx / RV_MAXC, c = idx % RV_MAXC;
    double v = 0.0;
    if (c < nco) {
      const int sv = src[c] >> 1;
      v = sigma[i] * ((src[c] & 1) ? yi[i + (int64_t)sv * ldy] : yr[i + (int64_t)sv * ldy]);
    }
    coef[idx] = v;
  }
}

// one pass over W for compact columns [c0, c0 + NC); RB rows per thread
#ifndef RV_RB
#define RV_RB 2
#endif
// launch shape of ritz_vectors_kernel (RV_RB rows per thread, RV_MINB CTAs per SM, columns unrolled RV_UNR):
// C5 (10 GB read) 2.41 ms at (2, 3, 4) -> 2.12 ms at (2, 2, 8), 0.74 of the measured HBM bandwidth
// (tools/ab_ritz.sh; RB 1/4, MINB 1/4-8 and UNR 12/16 slower)
#ifndef RV_MINB
#define RV_MINB 2
#endif
#ifndef RV_UNR
#define RV_UNR 8
#endif
constexpr int kRvUnr = RV_UNR;
template <int NC, int RB>
__device__ __forceinline__ void ritz_body(const double* __restrict__ W, int64_t ld, int64_t off, int64_t n, int nc,
                                          const double* __restrict__ cs, const int* __restrict__ dst, int c0,
                                          int nco, double* __restrict__ Xr, double* __restrict__ Xi, int64_t ldx,
                                          int64_t xoff) {
  const int64_t rpb = (int64_t)blockDim.x * RB;
  for (int64_t base = blockIdx.x * rpb; base < n; base += (int64_t)gridDim.x * rpb) {
    int64_t p[RB];
    bool ok[RB];
    double acc[RB][NC];
#pragma unroll
    for (int r = 0; r < RB; ++r) {
      p[r] = base + threadIdx.x + (int64_t)r * blockDim.x;
      ok[r] = p[r] < n;
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[r][c] = 0.0;
    }
    const double* wp = W + off;
#pragma unroll (kRvUnr)
    for (int i = 0; i < nc; ++i) {
      double w[RB];
#pragma unroll
      for (int r = 0; r < RB; ++r) w[r] = ok[r] ? __ldg(wp + p[r] + (int64_t)i * ld) : 0.0;
      const double2* ci = reinterpret_cast<const double2*>(cs + i * RV_MAXC + c0);
#pragma unroll
      for (int c2 = 0; c2 < NC / 2; ++c2) {
        const double2 cv = ci[c2];
#pragma unroll
        for (int r = 0; r < RB; ++r) {
          acc[r][2 * c2] = fma(cv.x, w[r], acc[r][2 * c2]);
          acc[r][2 * c2 + 1] = fma(cv.y, w[r], acc[r][2 * c2 + 1]);
        }
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      if (c0 + c >= nco) break;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int d = dst[2 * (c0 + c) + e];
        if (d == 0) continue;
        const int o = (d > 0 ? d : -d) - 1;
        double* out = ((o & 1) ? Xi : Xr) + xoff + (int64_t)(o >> 1) * ldx;
        const double sg = d > 0 ? 1.0 : -1.0;
#pragma unroll
        for (int r = 0; r < RB; ++r)
          if (ok[r]) out[p[r]] = sg * acc[r][c];
      }
    }
  }
}

__global__ void __launch_bounds__(256, RV_MINB) ritz_vectors_kernel(const double* __restrict__ W, int64_t ld, int64_t off,
                                                              int64_t n, int nc, const double* __restrict__ coef,
                                                              const int* __restrict__ meta, double* __restrict__ Xr,
                                                              double* __restrict__ Xi, int64_t ldx, int64_t xoff) {
  extern __shared__ double cs[];  // [nc][RV_MAXC]
  __shared__ int dst[2 * RV_MAXC];
  for (int t = threadIdx.x; t < nc * RV_MAXC; t += blockDim.x) cs[t] = coef[t];
  if (threadIdx.x < 2 * RV_MAXC) dst[threadIdx.x] = meta[1 + threadIdx.x];
  const int nco = meta[0];
  __syncthreads();
  // C5's ten Ritz vectors need 10-12 compact columns: one pass; more columns take more passes
  for (int c0 = 0; c0 < nco; c0 += 12) {
    if (nco - c0 <= 4)
      ritz_body<4, RV_RB>(W, ld, off, n, nc, cs, dst, c0, nco, Xr, Xi, ldx, xoff);
    else
      ritz_body<12, RV_RB>(W, ld, off, n, nc, cs, dst, c0, nco, Xr, Xi, ldx, xoff);
  }
}

// out[:, i] = sigma_i W[off:off+n, i]   (normalised basis columns, ld = ldo)
__global__ void scale_cols_kernel(const double* __restrict__ W, int64_t ld, int64_t off, int64_t n, int nc,
                                  const double* __restrict__ sigma, double* __restrict__ out, int64_t ldo) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < n * nc;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t p = idx % n;
    const int i = (int)(idx / n);
    out[p + (int64_t)i * ldo] = sigma[i] * W[off + p + (int64_t)i * ld];
  }
}

// partials[b][v][0..1] = sum ||(A - theta) x||^2, ||x||^2 for complex x = xr + i xi
__global__ void complex_residual_kernel(int64_t n, const double* __restrict__ Axr, const double* __restrict__ Axi,
                                        const double* __restrict__ xr, const double* __restrict__ xi, int64_t ldx,
                                        int64_t ldax, int nvec, const double* __restrict__ thr,
                                        const double* __restrict__ thi, double* __restrict__ partials) {
  __shared__ double red[64];
  for (int v = 0; v < nvec; ++v) {
    const double a = thr[v], b = thi[v];
    double s_res = 0.0, s_x = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
      const double r0 = xr[p + v * ldx], i0 = xi[p + v * ldx];
      const double rr = Axr[p + v * ldax] - a * r0 + b * i0;
      const double ri = Axi[p + v * ldax] - a * i0 - b * r0;
      s_res += rr * rr + ri * ri;
      s_x += r0 * r0 + i0 * i0;
    }
    double t[2] = {s_res, s_x}, o[2];
    block_sum_n<2>(t, red, o);
    if (threadIdx.x == 0) {
      partials[((int64_t)blockIdx.x * nvec + v) * 2 + 0] = o[0];
      partials[((int64_t)blockIdx.x * nvec + v) * 2 + 1] = o[1];
    }
  }
}

// out[c] = sum_b part[b*stride + c], c < ncomp (fixed order)
__global__ void sum_partials_kernel(const double* __restrict__ part, int grid, int stride, int ncomp,
                                    double* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncomp) return;
  double t = 0.0;
  for (int b = 0; b < grid; ++b) t += part[(int64_t)b * stride + c];
  out[c] = t;
}

__global__ void ctrl_reset_kernel(CtrlBlock* c, double thr, double fnorm) {
  c->stop_col = 0x7fffffff;
  c->breakdown = 0;
  c->exit_cols = 0;
  c->qr_cols = 0;
  c->rank_def = 0;
  c->rnorm = 0.0;
  c->fnorm = fnorm;
  c->thr = thr;
  c->cond = 0.0;
  c->r_est_last = 0.0;
}

// global column index -> index into the all-gathered vector [rank][maxn]
__global__ void remap_cols_kernel(int64_t nnz, const int32_t* __restrict__ cg, int32_t* __restrict__ co,
                                  int nranks, const int64_t* __restrict__ rb, int64_t maxn) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t g = cg[p];
    int r = 0;
    while (r + 1 < nranks && g >= rb[r + 1]) ++r;
    co[p] = (int32_t)(r * maxn + (g - rb[r]));
  }
}

// ------------------------------------------------------------------------------
cudaError_t launch_form_cols(int mode, const double* SW, int s, int j0, int J, int k, const double* H, int ldH,
                             const double* sigma, const double* gam, double* X, int64_t ldq, int64_t ldj,
                             cudaStream_t st) {
  const int tot = s * J;
  form_cols_kernel<<<(tot + 255) / 256, 256, 0, st>>>(mode, SW, s, j0, J, k, H, ldH, sigma, gam, X, ldq, ldj);
  return cudaGetLastError();
}

cudaError_t launch_utx(const double* U, int ldu, int s, int j0, const double* X, int J, double* Z, double* T,
                       int ldT, int tc0, int tacc, double* ws, int* cnt, cudaStream_t st) {
  if (j0 <= 0) return cudaSuccess;
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.A = U;
  g.sAm = ldu;
  g.sAk = 1;
  g.B = X;
  g.M = j0;
  g.J = J;
  g.K = s;
  g.mode = 0;
  g.Z = Z;
  g.T = T;
  g.ldT = ldT;
  g.tc0 = tc0;
  g.tacc = tacc;
  return launch_bgs_gemm(g, true, ws, cnt, st);
}

cudaError_t launch_xmuz(const double* U, int ldu, int s, int j0, double* X, int J, const double* Z, double* ws,
                        int* cnt, cudaStream_t st) {
  if (j0 <= 0) return cudaSuccess;
  GemmArgs g;
  memset(&g, 0, sizeof(g));
  g.A = U;
  g.sAm = 1;
  g.sAk = ldu;
  g.B = Z;
  g.M = s;
  g.J = J;
  g.K = j0;
  g.mode = 1;
  g.X = X;
  return launch_bgs_gemm(g, false, ws, cnt, st);
}

size_t panel_smem(int s, int J) { return sizeof(double) * ((size_t)s * (J + 1) + s); }

cudaError_t launch_panel(double* X, int s, int J, int j0, double* U, int ldu, double* T, int ldT, double* rvec,
                         double* rho, double* rest, CtrlBlock* ctrl, int track_res, int max_cols,
                         cudaStream_t st) {
  const size_t smem = panel_smem(s, J);
  cudaError_t e = set_smem_attr(panel_kernel, smem);
  if (e != cudaSuccess) return e;
  panel_kernel<<<1, 1024, smem, st>>>(X, s, J, j0, U, ldu, T, ldT, rvec, rho, rest, ctrl, track_res, max_cols);
  return cudaGetLastError();
}

cudaError_t launch_trsv(const double* T, int ldT, int n, const double* b, const double* scale, double* yout,
                        double* out, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  trsv_upper_kernel<<<1, CN_T, sizeof(double) * n, st>>>(T, ldT, n, b, scale, yout, out);
  return cudaGetLastError();
}

cudaError_t launch_cond(const double* T, int ldT, int n, int iters, CtrlBlock* ctrl, double* out,
                        cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  cond_kernel<<<1, CN_T, sizeof(double) * 2 * n, st>>>(T, ldT, n, iters, ctrl, out);
  return cudaGetLastError();
}

cudaError_t launch_assemble(double* x, const double* W, int64_t ld, int64_t off, int64_t n, const double* coef,
                            const int* ncp, int nc_max, int num_sms, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((n / 2 + 255) / 256 + 1, (int64_t)num_sms * 8);
  assemble_kernel<<<grid, 256, sizeof(double) * std::max(nc_max, 1), st>>>(x, W, ld, off, n, coef, ncp, nc_max);
  return cudaGetLastError();
}

size_t ritz_coef_doubles(int nc) { return (size_t)nc * RV_MAXC + 64; }

cudaError_t launch_ritz_vectors(const double* W, int64_t ld, int64_t off, int64_t n, int nc, const double* sigma,
                                const double* yr, const double* yi, int ldy, const double* th_re,
                                const double* th_im, const int* nsel, int nmax, double* work, double* Xr,
                                double* Xi, int64_t ldx, int64_t xoff, int num_sms, cudaStream_t st) {
  double* coef = work;
  int* meta = reinterpret_cast<int*>(work + (size_t)nc * RV_MAXC);
  ritz_coef_kernel<<<1, 256, 0, st>>>(sigma, yr, yi, ldy, nc, th_re, th_im, nsel, nmax, coef, meta);
  const size_t smem = sizeof(double) * (size_t)nc * RV_MAXC;
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(ritz_vectors_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return cudaGetLastError();
  int grid = (int)std::min<int64_t>((n + 256 * RV_RB - 1) / (256 * RV_RB), (int64_t)num_sms * RV_MINB);
  if (grid < 1) grid = 1;
  ritz_vectors_kernel<<<grid, 256, smem, st>>>(W, ld, off, n, nc, coef, meta, Xr, Xi, ldx, xoff);
  return cudaGetLastError();
}

cudaError_t launch_scale_cols(const double* W, int64_t ld, int64_t off, int64_t n, int nc, const double* sigma,
                              double* out, int64_t ldo, cudaStream_t st) {
  int64_t tot = n * nc;
  int grid = (int)std::min<int64_t>((tot + 255) / 256, 4096);
  if (grid < 1) grid = 1;
  scale_cols_kernel<<<grid, 256, 0, st>>>(W, ld, off, n, nc, sigma, out, ldo);
  return cudaGetLastError();
}

cudaError_t launch_complex_residual(int64_t n, const double* Axr, const double* Axi, const double* xr,
                                    const double* xi, int64_t ldx, int64_t ldax, int nvec, const double* thr,
                                    const double* thi, double* partials, int grid, cudaStream_t st) {
  complex_residual_kernel<<<grid, 256, 0, st>>>(n, Axr, Axi, xr, xi, ldx, ldax, nvec, thr, thi, partials);
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(const double* part, int grid, int stride, int ncomp, double* out, cudaStream_t st) {
  sum_partials_kernel<<<(ncomp + 127) / 128, 128, 0, st>>>(part, grid, stride, ncomp, out);
  return cudaGetLastError();
}

cudaError_t launch_ctrl_reset(CtrlBlock* c, double thr, double fnorm, cudaStream_t st) {
  ctrl_reset_kernel<<<1, 1, 0, st>>>(c, thr, fnorm);
  return cudaGetLastError();
}

cudaError_t launch_remap_cols(int64_t nnz, const int32_t* ci_global, int32_t* ci_out, int nranks,
                              const int64_t* rb_dev, int64_t maxn, cudaStream_t st) {
  int grid = (int)std::min<int64_t>((nnz + 255) / 256, 8192);
  if (grid < 1) grid = 1;
  remap_cols_kernel<<<grid, 256, 0, st>>>(nnz, ci_global, ci_out, nranks, rb_dev, maxn);
  return cudaGetLastError();
}

}  // namespace sks
