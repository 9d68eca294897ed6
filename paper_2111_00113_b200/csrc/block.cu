// block.cu -- block Krylov sRR: the block Chebyshev recurrence of Sec. "Block Chebyshev
// recurrence" on the matrix-free stencils, the sketched A B it implies, and the small multi-RHS
// triangular solve of the dense sRR matrix Mhat = T^-1 U^T S A B (Eq. Mhat-form).
//
//   B_1 = Omega,  B_2 = (2 rho)^-1 (A - cI) B_1,  B_j = rho^-1 [(A - cI) B_{j-1} - e B_{j-2}],
//   e = (dx^2 - dy^2) / (4 rho)
//
// One launch forms one block (b columns): no inner products and no reductions between the columns of a block or
// between blocks ("the lack of inner products ... evade communication and synchronization costs"), so
// a block is a pure streaming pass: read B_{j-1} (stencil) and B_{j-2}, write B_j -- 24 bytes per row and column.
// The kernel marches along the slowest grid axis (y in 2D, z in 3D) with the two previous planes of its column in
// registers; the in-plane neighbours come through L1 (they were loaded as plane centres by the neighbouring
// threads).  Columns use the basis layout of api.cu (ghost planes zero at a Dirichlet boundary, filled by the halo
// exchange between ranks).
#include <cstring>

#include "common.cuh"
#include "internal.h"

namespace sks {

constexpr int BK_TX = 128;   // threads per CTA along x
constexpr int BK_TY = 2;     // 3D: y rows per CTA (2D: 1)
constexpr int BK_ZCH = 32;   // planes per CTA march

struct BlockArgs {
  const double* in1;  // column i at in1 + i*ld (first interior point at + off)
  const double* in2;  // may be null
  double* out;
  int64_t ld, off, plane, m, nz;
  int dim;
  double cc, cm, cp;  // stencil: centre, minus neighbours, plus neighbours (reading O18)
  double alpha, shift, gamma;  // out = alpha (A - shift I) in1 + gamma in2
};

__global__ void __launch_bounds__(BK_TX * BK_TY) block_cheb_kernel(BlockArgs a) {
  const int col = blockIdx.z;
  const double* __restrict__ u = a.in1 + (int64_t)col * a.ld + a.off;
  const double* __restrict__ v = a.in2 ? a.in2 + (int64_t)col * a.ld + a.off : nullptr;
  double* __restrict__ o = a.out + (int64_t)col * a.ld + a.off;
  const int m = (int)a.m;
  const int x = blockIdx.x * BK_TX + threadIdx.x;
  int y = 0;
  if (a.dim == 3) y = blockIdx.y / ((a.nz + BK_ZCH - 1) / BK_ZCH) * BK_TY + threadIdx.y;
  const int zc = (a.dim == 3) ? (int)(blockIdx.y % ((a.nz + BK_ZCH - 1) / BK_ZCH)) : (int)blockIdx.y;
  const int z0 = zc * BK_ZCH, z1 = min((int)a.nz, z0 + BK_ZCH);
  if (x >= m || y >= m || z0 >= z1) return;
  const int64_t pl = a.plane;
  const int64_t c0 = (a.dim == 3) ? (int64_t)y * m + x : x;  // in-plane offset
  const bool xl = x > 0, xr = x < m - 1, yl = a.dim == 3 && y > 0, yr = a.dim == 3 && y < m - 1;
  // march along the slowest axis: the ghost planes (-1 and nz) hold zeros or the neighbour rank's planes;
  // BK_U planes per iteration with all their loads issued before any use (memory-level parallelism)
  constexpr int BK_U = 4;
  double um = __ldg(u + c0 + (int64_t)(z0 - 1) * pl);
  double uc = __ldg(u + c0 + (int64_t)z0 * pl);
  for (int zb = z0; zb < z1; zb += BK_U) {
    double up[BK_U], xm[BK_U], xp[BK_U], ym[BK_U], yp[BK_U], vv[BK_U];
#pragma unroll
    for (int i = 0; i < BK_U; ++i) {
      const int z = zb + i;
      const bool ok = z < z1;
      const double* uz = u + c0 + (int64_t)z * pl;
      up[i] = ok ? __ldg(uz + pl) : 0.0;
      xm[i] = (ok && xl) ? __ldg(uz - 1) : 0.0;
      xp[i] = (ok && xr) ? __ldg(uz + 1) : 0.0;
      ym[i] = (ok && yl) ? __ldg(uz - m) : 0.0;
      yp[i] = (ok && yr) ? __ldg(uz + m) : 0.0;
      vv[i] = (ok && v) ? __ldg(v + c0 + (int64_t)z * pl) : 0.0;
    }
#pragma unroll
    for (int i = 0; i < BK_U; ++i) {
      const int z = zb + i;
      if (z < z1) {
        const double sm = um + xm[i] + ym[i];
        const double sp = up[i] + xp[i] + yp[i];
        const double Au = a.cc * uc + a.cm * sm + a.cp * sp;
        double r = a.alpha * (Au - a.shift * uc);
        if (v) r += a.gamma * vv[i];
        o[c0 + (int64_t)z * pl] = r;
        um = uc;
        uc = up[i];
      }
    }
  }
}

cudaError_t launch_block_cheb(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off, int64_t ld, double cc,
                              double cm, double cp, const double* in1, const double* in2, double* out, int ncols,
                              double alpha, double shift, double gamma, cudaStream_t st) {
  if (ncols <= 0 || nz <= 0) return cudaSuccess;
  BlockArgs a;
  a.in1 = in1;
  a.in2 = in2;
  a.out = out;
  a.ld = ld;
  a.off = off;
  a.plane = plane;
  a.m = m;
  a.nz = nz;
  a.dim = dim;
  a.cc = cc;
  a.cm = cm;
  a.cp = cp;
  a.alpha = alpha;
  a.shift = shift;
  a.gamma = gamma;
  const int zch = (int)((nz + BK_ZCH - 1) / BK_ZCH);
  dim3 grid((unsigned)((m + BK_TX - 1) / BK_TX), 1, (unsigned)ncols);
  dim3 block(BK_TX, dim == 3 ? BK_TY : 1);
  grid.y = (dim == 3) ? (unsigned)(((m + BK_TY - 1) / BK_TY) * zch) : (unsigned)zch;
  block_cheb_kernel<<<grid, block, 0, st>>>(a);
  return cudaGetLastError();
}

// S A B from the sketched block columns through the recurrence (reading O34):
//   A B_1 = 2 rho B_2 + c B_1,  A B_j = rho B_{j+1} + c B_j + e B_{j-1}  (j >= 2)
// SW: s x ((p+1) b) column-major (ld s); SAB: s x (p b) column-major (ld s).
__global__ void block_sab_kernel(const double* __restrict__ SW, int s, int b, int p, double rho, double c, double e,
                                 double* __restrict__ SAB) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t tot = (int64_t)s * b * p;
  if (idx >= tot) return;
  const int q = (int)(idx % s);
  const int col = (int)(idx / s);  // (j-1) b + i
  const int j = col / b + 1, i = col % b;
  double r;
  if (j == 1) {
    r = 2.0 * rho * SW[(int64_t)(b + i) * s + q] + c * SW[(int64_t)i * s + q];
  } else {
    r = rho * SW[(int64_t)(j * b + i) * s + q] + c * SW[(int64_t)((j - 1) * b + i) * s + q] +
        e * SW[(int64_t)((j - 2) * b + i) * s + q];
  }
  SAB[(int64_t)col * s + q] = r;
}

cudaError_t launch_block_sab(const double* SW, int s, int b, int p, double rho, double c, double e, double* SAB,
                             cudaStream_t st) {
  const int64_t tot = (int64_t)s * b * p;
  block_sab_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(SW, s, b, p, rho, c, e, SAB);
  return cudaGetLastError();
}

// X <- T^-1 X for nrhs right-hand sides (T n x n upper triangular, ld ldT; X n x nrhs, ld ldx): one CTA per
// column, column-oriented back substitution (x_i = x_i / T_ii, then x_l -= T_li x_i for l < i).
__global__ void __launch_bounds__(256) trsm_upper_kernel(const double* __restrict__ T, int ldT, int n, double* X,
                                                         int ldx) {
  extern __shared__ double xs[];
  double* x = X + (int64_t)blockIdx.x * ldx;
  for (int i = threadIdx.x; i < n; i += blockDim.x) xs[i] = x[i];
  __syncthreads();
  for (int i = n - 1; i >= 0; --i) {
    const double xi = xs[i] / T[i + (int64_t)i * ldT];
    __syncthreads();  // every thread has read xs[i]
    if (threadIdx.x == 0) xs[i] = xi;
    for (int l = threadIdx.x; l < i; l += blockDim.x) xs[l] -= T[l + (int64_t)i * ldT] * xi;
    __syncthreads();
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = xs[i];
}

cudaError_t launch_trsm_upper(const double* T, int ldT, int n, double* X, int ldx, int nrhs, cudaStream_t st) {
  if (n <= 0 || nrhs <= 0) return cudaSuccess;
  const size_t smem = sizeof(double) * (size_t)n;
  if (smem > 48 * 1024) {
    if (cudaError_t e = set_smem_attr(trsm_upper_kernel, smem)) return e;
  }
  trsm_upper_kernel<<<nrhs, 256, smem, st>>>(T, ldT, n, X, ldx);
  return cudaGetLastError();
}

// V = I (n x n, ld ldv) and sigma[0..nc) = 1
__global__ void eye_ones_kernel(double* V, int n, int ldv, double* sigma, int nc) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (V && idx < (int64_t)n * n) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    V[i + (int64_t)j * ldv] = (i == j) ? 1.0 : 0.0;
  }
  if (sigma && idx < nc) sigma[idx] = 1.0;
}

cudaError_t launch_eye_ones(double* V, int n, int ldv, double* sigma, int nc, cudaStream_t st) {
  const int64_t tot = std::max<int64_t>(V ? (int64_t)n * n : 0, nc);
  if (tot <= 0) return cudaSuccess;
  eye_ones_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(V, n, ldv, sigma, nc);
  return cudaGetLastError();
}

// ---- deferred Chebyshev bookkeeping (see StepArgs::defer): the per-column partial sums of a
// batch, reduced in a fixed order to SKS_NP scalars per column (then all-reduced once per batch at P > 1) ...
__global__ void cheb_colsum_kernel(const double* __restrict__ part, int grid, int pstride, int j0, int j1,
                                   double* __restrict__ sums) {
  const int j = j0 + blockIdx.x;
  if (j >= j1) return;
  const double* p = part + (int64_t)j * pstride * SKS_NP;
  for (int i = threadIdx.x; i < SKS_NP; i += blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < grid; ++b) t += p[(int64_t)b * SKS_NP + i];
    sums[(int64_t)j * SKS_NP + i] = t;
  }
}

// ... and the recurrence bookkeeping of columns [j0, j1) in order, exactly what step_prologue does for one column
// (A b_j = gam_j w_{j+1} + sum_l H[l, j] b_l; sigma_j = 1/||w_j||; breakdown, reading O10)
__global__ void cheb_finalize_kernel(const double* __restrict__ sums, int j0, int j1, double rho, double c0, double e,
                                     double* sigma, double* H, int ldH, double* mnorm, double* gam, CtrlBlock* ctrl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  for (int jm = j0; jm < j1; ++jm) {
    if (ctrl->stop_col <= jm) return;
    const double N = sums[(int64_t)jm * SKS_NP + 0];
    const double nu = sqrt(N);
    const double ref = 1.0 / sigma[jm - 1];  // the previous raw vector's norm
    if (!(N > 0.0) || !isfinite(N) || nu <= 1e-14 * ref) {
      ctrl->stop_col = jm;
      ctrl->breakdown = 1;
      H[jm + (int64_t)(jm - 1) * ldH] = gam[jm - 1] * nu;
      return;
    }
    const double sg = 1.0 / nu;
    const double al = 1.0 / rho;  // alpha of launch jm + 1 (jm >= 2)
    gam[jm] = sg / al;
    H[jm + (int64_t)jm * ldH] = c0;                                   // -beta_u / alpha
    H[(jm - 1) + (int64_t)jm * ldH] = -sg * (-e / rho) / (al * sigma[jm - 1]);
    sigma[jm] = sg;
    mnorm[jm] = sg * sqrt(sums[(int64_t)jm * SKS_NP + 2]);
    H[jm + (int64_t)(jm - 1) * ldH] = gam[jm - 1] * nu;
  }
}

cudaError_t launch_cheb_colsum(const double* part, int grid, int pstride, int j0, int j1, double* sums,
                               cudaStream_t st) {
  if (j1 <= j0) return cudaSuccess;
  cheb_colsum_kernel<<<j1 - j0, 32, 0, st>>>(part, grid, pstride, j0, j1, sums);
  return cudaGetLastError();
}

cudaError_t launch_cheb_finalize(const double* sums, int j0, int j1, double rho, double c0, double e, double* sigma,
                                 double* H, int ldH, double* mnorm, double* gam, CtrlBlock* ctrl, cudaStream_t st) {
  if (j1 <= j0) return cudaSuccess;
  cheb_finalize_kernel<<<1, 32, 0, st>>>(sums, j0, j1, rho, c0, e, sigma, H, ldH, mnorm, gam, ctrl);
  return cudaGetLastError();
}

// ---- whitening (Fact "Whitening" P:598-612; reading O36) ---------------------------
// Wn[:, i] = sum_{l <= i} W[:, l] Z[l, i] for i < J (Z = diag(sigma) T_J^{-1}, upper triangular), interior rows of
// the basis layout (pitch ld, first interior point at off), into a separate buffer with the same layout; per
// (row-block group, column) sums of squares of the outputs in part[blockIdx.y][i] (fixed-order, no atomics).
constexpr int WG_R = 64, WG_C = 32, WG_K = 32;
__global__ void __launch_bounds__(256) whiten_gemm_kernel(const double* __restrict__ W, int64_t ld, int64_t off,
                                                          int64_t n, int J, const double* __restrict__ Z, int ldz,
                                                          double* __restrict__ Wn, double* __restrict__ part) {
  __shared__ double As[WG_K][WG_R + 1];
  __shared__ double Bs[WG_K][WG_C + 1];
  const int tid = threadIdx.x, lane = tid & 31, cg = tid >> 5;  // rows lane, lane + 32; columns 4 cg .. 4 cg + 3
  const int i0 = blockIdx.x * WG_C;
  double ss[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t rb = blockIdx.y; rb * WG_R < n; rb += gridDim.y) {
    const int64_t r0 = rb * WG_R;
    double acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
    const int lend = min(J, i0 + WG_C);  // Z[l, i] = 0 for l > i
    for (int l0 = 0; l0 < lend; l0 += WG_K) {
      __syncthreads();
      for (int e = tid; e < WG_K * WG_R; e += 256) {
        const int l = e / WG_R, r = e - l * WG_R;
        As[l][r] = (l0 + l < J && r0 + r < n) ? W[(int64_t)(l0 + l) * ld + off + r0 + r] : 0.0;
      }
      for (int e = tid; e < WG_K * WG_C; e += 256) {
        const int l = e / WG_C, c = e - l * WG_C;
        const int gl = l0 + l, gi = i0 + c;
        Bs[l][c] = (gl < J && gi < J && gl <= gi) ? Z[gl + (int64_t)gi * ldz] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int l = 0; l < WG_K; ++l) {
        const double a0 = As[l][lane], a1 = As[l][lane + 32];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double z = Bs[l][4 * cg + b];
          acc[0][b] = fma(a0, z, acc[0][b]);
          acc[1][b] = fma(a1, z, acc[1][b]);
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int64_t r = r0 + lane + 32 * a;
      if (r < n) {
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const int i = i0 + 4 * cg + b;
          if (i < J) {
            Wn[(int64_t)i * ld + off + r] = acc[a][b];
            ss[b] = fma(acc[a][b], acc[a][b], ss[b]);
          }
        }
      }
    }
  }
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    double v = ss[b];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int i = i0 + 4 * cg + b;
    if (lane == 0 && i < J) part[(int64_t)blockIdx.y * J + i] = v;
  }
}

// sums[i] = sum over the row-block groups of part[g][i], fixed order
__global__ void colsum_kernel(const double* __restrict__ part, int ng, int J, double* __restrict__ sums) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= J) return;
  double t = 0.0;
  for (int g = 0; g < ng; ++g) t += part[(int64_t)g * J + i];
  sums[i] = t;
}

// after the whitening: sigma_i = 1/||Wn_i|| (unit basis columns, reading O36), T[:J, :J] = diag(sigma), the
// control block continues at J QR'd columns
__global__ void whiten_finish_kernel(const double* __restrict__ sums, int J, double* sigma, double* T, int ldT,
                                     CtrlBlock* ctrl) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx < (int64_t)J * J) {
    const int i = (int)(idx % J), j = (int)(idx / J);
    T[i + (int64_t)j * ldT] = (i == j) ? 1.0 / sqrt(sums[i]) : 0.0;
  }
  if (idx < J) sigma[idx] = 1.0 / sqrt(sums[idx]);
  if (idx == 0) {
    ctrl->qr_cols = J;
    ctrl->cond = 0.0;
    ctrl->exit_cols = 0;
  }
}

// Z[l, i] *= sigma[l]  (Z = diag(sigma) T^{-1})
__global__ void scale_rows_kernel(double* Z, int J, int ldz, const double* __restrict__ sigma) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)J * J) return;
  const int l = (int)(idx % J), i = (int)(idx / J);
  Z[l + (int64_t)i * ldz] *= sigma[l];
}

// partial sums the step after a whitening needs (step_prologue of launch J, the whitened column J-1 as w_{J-1}):
// [0] ||u||^2, [1] <u, A u>, [2] ||A u||^2, [3 + slot_l] <v_l, A u>; stencil operator, ghost planes valid
struct WpArgs {
  const double* u;
  const double* v[SKS_KMAX];
  int slot[SKS_KMAX];
  int nv;
  int64_t n, plane, m;
  int dim;
  double cc, cm, cp;
  double* part;  // [gridDim.x][SKS_NP]
};
__global__ void __launch_bounds__(256) whiten_partials_kernel(WpArgs a) {
  double acc[3 + SKS_KMAX];
#pragma unroll
  for (int i = 0; i < 3 + SKS_KMAX; ++i) acc[i] = 0.0;
  const int64_t m = a.m;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < a.n; idx += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = idx / a.plane, ip = idx - z * a.plane;
    const int64_t x = (a.dim == 3) ? ip % m : ip, y = (a.dim == 3) ? ip / m : 0;
    const double* u = a.u + idx;
    double sm = u[-a.plane] + (x > 0 ? u[-1] : 0.0);
    double sp = u[a.plane] + (x < m - 1 ? u[1] : 0.0);
    if (a.dim == 3) {
      sm += (y > 0) ? u[-m] : 0.0;
      sp += (y < m - 1) ? u[m] : 0.0;
    }
    const double uc = u[0];
    const double Au = a.cc * uc + a.cm * sm + a.cp * sp;
    acc[0] = fma(uc, uc, acc[0]);
    acc[1] = fma(uc, Au, acc[1]);
    acc[2] = fma(Au, Au, acc[2]);
    for (int l = 0; l < a.nv; ++l) acc[3 + l] = fma(a.v[l][idx], Au, acc[3 + l]);
  }
  __shared__ double red[(3 + SKS_KMAX) * 32];
  __shared__ double R[3 + SKS_KMAX];
  block_sum_n<3 + SKS_KMAX>(acc, red, R);
  if (threadIdx.x == 0) {
    double out[SKS_NP];
    for (int i = 0; i < SKS_NP; ++i) out[i] = 0.0;
    out[0] = R[0];
    out[1] = R[1];
    out[2] = R[2];
    for (int l = 0; l < a.nv; ++l)
      if (a.slot[l] >= 3 && a.slot[l] < SKS_NP) out[a.slot[l]] = R[3 + l];
    for (int i = 0; i < SKS_NP; ++i) a.part[(int64_t)blockIdx.x * SKS_NP + i] = out[i];
  }
}

// r = g - U[:, :J] rho[:J]  (the explicit sketched residual vector of the QR, reading O12)
__global__ void resid_restore_kernel(double* __restrict__ r, const double* __restrict__ g, const double* __restrict__ U,
                                     int ldu, const double* __restrict__ rho, int J, int s) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= s) return;
  double t = g[q];
  for (int i = 0; i < J; ++i) t -= U[q + (int64_t)i * ldu] * rho[i];
  r[q] = t;
}

cudaError_t launch_resid_restore(double* r, const double* g, const double* U, int ldu, const double* rho, int J, int s,
                                 cudaStream_t st) {
  resid_restore_kernel<<<(s + 127) / 128, 128, 0, st>>>(r, g, U, ldu, rho, J, s);
  return cudaGetLastError();
}

cudaError_t launch_whiten_gemm(const double* W, int64_t ld, int64_t off, int64_t n, int J, const double* Z, int ldz,
                               double* Wn, double* part, int ngroups, cudaStream_t st) {
  if (J <= 0) return cudaSuccess;
  whiten_gemm_kernel<<<dim3((unsigned)((J + WG_C - 1) / WG_C), (unsigned)ngroups), 256, 0, st>>>(W, ld, off, n, J, Z,
                                                                                                ldz, Wn, part);
  return cudaGetLastError();
}

cudaError_t launch_colsum(const double* part, int ng, int J, double* sums, cudaStream_t st) {
  colsum_kernel<<<(J + 127) / 128, 128, 0, st>>>(part, ng, J, sums);
  return cudaGetLastError();
}

cudaError_t launch_whiten_finish(const double* sums, int J, double* sigma, double* T, int ldT, CtrlBlock* ctrl,
                                 cudaStream_t st) {
  const int64_t tot = std::max<int64_t>((int64_t)J * J, 1);
  whiten_finish_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(sums, J, sigma, T, ldT, ctrl);
  return cudaGetLastError();
}

cudaError_t launch_scale_rows(double* Z, int J, int ldz, const double* sigma, cudaStream_t st) {
  const int64_t tot = (int64_t)J * J;
  if (tot <= 0) return cudaSuccess;
  scale_rows_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(Z, J, ldz, sigma);
  return cudaGetLastError();
}

cudaError_t launch_whiten_partials(const double* u, const double* const* v, const int* slot, int nv, int64_t n,
                                   int64_t plane, int64_t m, int dim, double cc, double cm, double cp, double* part,
                                   int grid, cudaStream_t st) {
  WpArgs a;
  memset(&a, 0, sizeof(a));
  a.u = u;
  a.nv = nv;
  for (int l = 0; l < nv && l < SKS_KMAX; ++l) {
    a.v[l] = v[l];
    a.slot[l] = slot[l];
  }
  a.n = n;
  a.plane = plane;
  a.m = m;
  a.dim = dim;
  a.cc = cc;
  a.cm = cm;
  a.cp = cp;
  a.part = part;
  whiten_partials_kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sks

namespace sks {
// ---- 2D Chebyshev matrix-powers step (SURVEY NEXT(1) "depth-s halos"; Eq. Chebrecurse P:1192-1199 with the
// deferred bookkeeping of O37): S consecutive columns w_j .. w_{j+S-1} of the raw recurrence
//     w_i = rho^-1 [ (A - cI) w_{i-1} - e w_{i-2} ]
// in ONE launch.  CTA b owns the lines [y0, y1) of the slab; it stages w_{j-1}, w_{j-2} on the lines
// [y0 - S - 1, y1 + S + 1) in shared memory (ghost lines: Dirichlet zeros at the domain boundary, the neighbour
// rank's lines -- exchanged once per launch with depth G >= S + 1 -- inside), then computes step t on the lines
// [y0 - S + t, y1 + S - t) (the valid region shrinks by one line per step), writes its own lines of every column
// and their ||w||^2 partial into the per-column partial slots the deferred finalisation reduces.  Per S columns the
// two input columns are read once (plus 2 (S + 1) halo lines per CTA) and S columns written: about
// 8 (2 + 2 (2S+2) / lines_per_cta) / S + 8 bytes per row and column instead of 24.
struct MpkArgs {
  double* W;
  int64_t ld, off, m, nz, z0, mglob;
  double cc, cm, cp, rho, c0, e;
  int j, S, L;          // first column, columns, staged lines per buffer
  double* partc;        // partc + col * pstride * SKS_NP + cta * SKS_NP
  int pstride, zero_to; // rows [gridDim.x, zero_to) of each column's slot are zero-filled
  const CtrlBlock* ctrl;
};

__global__ void __launch_bounds__(256) cheb_mpk2d_kernel(MpkArgs a) {
  extern __shared__ double mk[];
  if (a.ctrl->stop_col < a.j || a.ctrl->exit_cols != 0) return;
  const int64_t m = a.m;
  const int b = blockIdx.x;
  const int y0 = (int)((a.nz * b) / gridDim.x), y1 = (int)((a.nz * (b + 1)) / gridDim.x);
  const int lb = y0 - a.S - 1;  // first staged line
  double* buf[3] = {mk, mk + (size_t)a.L * m, mk + (size_t)2 * a.L * m};
  double* U = buf[0];
  double* V = buf[1];
  double* Wn = buf[2];
  const double* gU = a.W + (int64_t)(a.j - 1) * a.ld + a.off;
  const double* gV = a.W + (int64_t)(a.j - 2) * a.ld + a.off;
  const int nl = y1 - y0 + 2 * a.S + 2;
  for (int64_t i = threadIdx.x; i < (int64_t)nl * m; i += blockDim.x) {
    const int l = (int)(i / m);
    const int64_t x = i - (int64_t)l * m;
    const int64_t row = (int64_t)(lb + l) * m + x;  // ghost lines are within [-G, nz + G)
    U[i] = gU[row];
    V[i] = gV[row];
  }
  __syncthreads();
  const double irho = 1.0 / a.rho;
  double nrm[8];
  for (int t = 0; t < 8; ++t) nrm[t] = 0.0;
  for (int t = 0; t < a.S; ++t) {
    const int la = y0 - a.S + t, lz = y1 + a.S - t;  // computed lines [la, lz)
    double* wcol = a.W + (int64_t)(a.j + t) * a.ld + a.off;
    double nt = 0.0;
    for (int64_t i = threadIdx.x; i < (int64_t)(lz - la) * m; i += blockDim.x) {
      const int l = la + (int)(i / m);
      const int64_t x = i - (int64_t)(l - la) * m;
      const int64_t k = (int64_t)(l - lb) * m + x;  // index in the staged buffers
      const int64_t gl = a.z0 + l;                   // global line
      double w = 0.0;
      if (gl >= 0 && gl < a.mglob) {
        const double u = U[k];
        const double sm = (x > 0 ? U[k - 1] : 0.0) + U[k - m];
        const double sp = (x < m - 1 ? U[k + 1] : 0.0) + U[k + m];
        const double Au = a.cc * u + a.cm * sm + a.cp * sp;
        w = (Au - a.c0 * u - a.e * V[k]) * irho;
      }
      Wn[k] = w;
      if (l >= y0 && l < y1) {
        wcol[(int64_t)l * m + x] = w;
        nt = fma(w, w, nt);
      }
    }
    nrm[t] = nt;
    __syncthreads();
    double* tmp = V;  // rotate: V <- U, U <- Wn, Wn <- old V
    V = U;
    U = Wn;
    Wn = tmp;
  }
  // per-column partial ||w||^2 of this CTA's lines (fixed-order block reduction)
  __shared__ double red[32 * 8];
  __shared__ double R[8];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  for (int t = 0; t < a.S; ++t) {
    const double v = warp_sum(nrm[t]);
    if (lane == 0) red[t * 32 + wid] = v;
  }
  __syncthreads();
  if (wid < a.S) {
    double v = lane < nw ? red[wid * 32 + lane] : 0.0;
    v = warp_sum(v);
    if (lane == 0) R[wid] = v;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < a.S * SKS_NP; i += blockDim.x) {
    const int t = i / SKS_NP, q = i - t * SKS_NP;
    a.partc[((size_t)(a.j + t) * a.pstride + b) * SKS_NP + q] = (q == 0) ? R[t] : 0.0;
  }
  if (b == 0)  // rows past this grid (the step kernels' grid is larger): zero, so the finaliser may sum them
    for (int i = threadIdx.x; i < a.S * (a.zero_to - (int)gridDim.x) * SKS_NP; i += blockDim.x) {
      const int per = (a.zero_to - (int)gridDim.x) * SKS_NP;
      const int t = i / per, r = i - t * per;
      a.partc[((size_t)(a.j + t) * a.pstride + gridDim.x) * SKS_NP + r] = 0.0;
    }
}

size_t mpk2d_smem(int64_t m, int64_t nz, int grid, int S) {
  const int64_t own = (nz + grid - 1) / grid;
  return sizeof(double) * 3 * (size_t)(own + 2 * S + 2) * m;
}

cudaError_t launch_cheb_mpk2d(double* W, int64_t ld, int64_t off, int64_t m, int64_t nz, int64_t z0, int64_t mglob,
                              double cc, double cm, double cp, double rho, double c0, double e, int j, int S,
                              double* partc, int pstride, int zero_to, const CtrlBlock* ctrl, int grid,
                              cudaStream_t st) {
  if (S < 1 || S > 8) return cudaErrorInvalidValue;
  MpkArgs a;
  a.W = W;
  a.ld = ld;
  a.off = off;
  a.m = m;
  a.nz = nz;
  a.z0 = z0;
  a.mglob = mglob;
  a.cc = cc;
  a.cm = cm;
  a.cp = cp;
  a.rho = rho;
  a.c0 = c0;
  a.e = e;
  a.j = j;
  a.S = S;
  a.L = (int)((nz + grid - 1) / grid + 2 * S + 2);
  a.partc = partc;
  a.pstride = pstride;
  a.zero_to = zero_to;
  a.ctrl = ctrl;
  const size_t smem = mpk2d_smem(m, nz, grid, S);
  if (cudaError_t err = set_smem_attr(cheb_mpk2d_kernel, smem)) return err;
  cheb_mpk2d_kernel<<<grid, 256, smem, st>>>(a);
  return cudaGetLastError();
}
}  // namespace sks
