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
  // march along the slowest axis: the ghost planes (-1 and nz) hold zeros or the neighbour rank's planes
  double um = __ldg(u + c0 + (int64_t)(z0 - 1) * pl);
  double uc = __ldg(u + c0 + (int64_t)z0 * pl);
  for (int z = z0; z < z1; ++z) {
    const double* uz = u + c0 + (int64_t)z * pl;
    const double up = __ldg(uz + pl);
    double sm = um + (xl ? __ldg(uz - 1) : 0.0);
    double sp = up + (xr ? __ldg(uz + 1) : 0.0);
    if (a.dim == 3) {
      sm += yl ? __ldg(uz - m) : 0.0;
      sp += yr ? __ldg(uz + m) : 0.0;
    }
    const double Au = a.cc * uc + a.cm * sm + a.cp * sp;
    double r = a.alpha * (Au - a.shift * uc);
    if (v) r += a.gamma * __ldg(v + c0 + (int64_t)z * pl);
    o[c0 + (int64_t)z * pl] = r;
    um = uc;
    uc = up;
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

}  // namespace sks
