// stencil.cu -- fused truncated-Arnoldi step for the matrix-free 5-/7-point
// convection-diffusion operators (reading O18), and plain y = A x.
//
// Vector layout in HBM: each column is a slab of
// (nz + 2G) planes x plane points, G = 2 ghost planes on each side (zero at the
// physical Dirichlet boundary, filled by the halo exchange at interior partition
// boundaries), column pitch ld (multiple of 64 doubles).  Interior points of a
// column are contiguous (offset G*plane), which the sketch kernel relies on.
#include "step.cuh"
#include "internal.h"

namespace sks {

// ------------------------------------------------------------------------------
// 2D: independent TX x TY output tiles, grid-stride over tiles.
//   sU : U (= w_{j-1}, x or v0) on the tile + 2-point halo
//   sV : the other window vectors on the tile + 1-point halo
//   sW : the new column w_j on the tile + 1-point halo (zero outside the domain)
// ------------------------------------------------------------------------------
constexpr int T2X = 64, T2Y = 16;
constexpr int E2X = T2X + 4, E2Y = T2Y + 4, E1X = T2X + 2, E1Y = T2Y + 2;

template <int KM>
__global__ void __launch_bounds__(256) step2d_kernel(StepArgs a) {
  extern __shared__ double sm[];
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  if (!step_prologue(a, &cf, red)) return;
  double* sU = sm;
  double* sW = sU + E2X * E2Y;
  double* sV = sW + E1X * E1Y;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t m = a.m, nz = a.nz, G = a.G, z0 = a.z0;
  const double cc = a.cc, cm = a.cm, cp = a.cp;
  const double alpha = cf.alpha, beta_u = cf.beta_u;
  const int nv = cf.nv;
  double* Wout = a.W + (int64_t)a.j * a.ld + a.off;
  if (a.mode != 0) Wout = a.W + a.off;
  const double* U = cf.U + a.off;
  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;

  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    const int64_t tx0 = (tile % a.tiles_x) * T2X;
    const int64_t ty0 = (tile / a.tiles_x) * T2Y;
    for (int idx = tid; idx < E2X * E2Y; idx += nt) {
      const int ex = idx % E2X, ey = idx / E2X;
      const int64_t x = tx0 - 2 + ex, ly = ty0 - 2 + ey;
      double v = 0.0;
      if (x >= 0 && x < m && ly >= -G && ly < nz + G) v = U[ly * m + x];
      sU[idx] = v;
    }
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) {
      if (l < nv) {
        const double* V = cf.V[l] + a.off;
        for (int idx = tid; idx < E1X * E1Y; idx += nt) {
          const int ex = idx % E1X, ey = idx / E1X;
          const int64_t x = tx0 - 1 + ex, ly = ty0 - 1 + ey;
          double v = 0.0;
          if (x >= 0 && x < m && ly >= -G && ly < nz + G) v = V[ly * m + x];
          sV[l * E1X * E1Y + idx] = v;
        }
      }
    }
    __syncthreads();
    for (int idx = tid; idx < E1X * E1Y; idx += nt) {
      const int ex = idx % E1X, ey = idx / E1X;
      const int64_t x = tx0 - 1 + ex, ly = ty0 - 1 + ey, gy = z0 + ly;
      double w = 0.0;
      if (x >= 0 && x < m && gy >= 0 && gy < m && ly >= 1 - G && ly < nz + G - 1) {
        const int c = (ey + 1) * E2X + ex + 1;
        const double u = sU[c];
        const double Au = cc * u + cm * (sU[c - 1] + sU[c - E2X]) + cp * (sU[c + 1] + sU[c + E2X]);
        w = alpha * Au + beta_u * u;
#pragma unroll
        for (int l = 0; l < KM - 1; ++l)
          if (l < nv) w += cf.c[l] * sV[l * E1X * E1Y + idx];
      }
      sW[idx] = w;
    }
    __syncthreads();
    for (int idx = tid; idx < T2X * T2Y; idx += nt) {
      const int ex = idx % T2X, ey = idx / T2X;
      const int64_t x = tx0 + ex, ly = ty0 + ey;
      if (x < m && ly < nz) {
        const int c = (ey + 1) * E1X + ex + 1;
        const double w = sW[c];
        const double Aw = cc * w + cm * (sW[c - 1] + sW[c - E1X]) + cp * (sW[c + 1] + sW[c + E1X]);
        Wout[ly * m + x] = w;
        acc[0] += w * w;
        acc[1] += w * Aw;
        acc[2] += Aw * Aw;
        if (cf.uslot >= 0) acc[KM + 2] += sU[(ey + 2) * E2X + ex + 2] * Aw;
#pragma unroll
        for (int l = 0; l < KM - 1; ++l)
          if (l < nv) acc[3 + l] += sV[l * E1X * E1Y + c] * Aw;
      }
    }
    __syncthreads();
  }
  step_epilogue<KM>(a, &cf, acc, red);
}

// ------------------------------------------------------------------------------
// 3D: (TX x TY) column tiles marching along z through a chunk of planes, with
// rolling plane buffers (U: 3 planes + 2-halo, W: 3 planes + 1-halo, V: 2 planes + 1-halo).
// ------------------------------------------------------------------------------
constexpr int T3X = 32, T3Y = 16;
constexpr int P2X = T3X + 4, P2Y = T3Y + 4, P1X = T3X + 2, P1Y = T3Y + 2;
constexpr int P2 = P2X * P2Y, P1 = P1X * P1Y;

template <int KM>
__global__ void __launch_bounds__(256) step3d_kernel(StepArgs a) {
  extern __shared__ double sm[];
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  if (!step_prologue(a, &cf, red)) return;
  double* sU = sm;             // [3][P2]
  double* sW = sU + 3 * P2;    // [3][P1]
  double* sV = sW + 3 * P1;    // [KM-1][2][P1]
  const int tid = threadIdx.x, nt = blockDim.x;
  const int64_t m = a.m, nz = a.nz, G = a.G, z0 = a.z0, pl = a.plane;
  const double cc = a.cc, cm = a.cm, cp = a.cp;
  const double alpha = cf.alpha, beta_u = cf.beta_u;
  const int nv = cf.nv;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;
  const double* U = cf.U + a.off;
  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;
  const int64_t nchunks = (nz + a.zchunk - 1) / a.zchunk;

  for (int64_t item = blockIdx.x; item < a.ntiles; item += gridDim.x) {
    const int64_t tcol = item % ((int64_t)a.tiles_x * a.tiles_y);
    const int64_t zc = item / ((int64_t)a.tiles_x * a.tiles_y);
    if (zc >= nchunks) continue;
    const int64_t tx0 = (tcol % a.tiles_x) * T3X, ty0 = (tcol / a.tiles_x) * T3Y;
    const int64_t zs = zc * a.zchunk, ze = min(nz, zs + (int64_t)a.zchunk);

    auto loadU = [&](int64_t lz) {
      double* dst = sU + (int)(((lz % 3) + 3) % 3) * P2;
      const bool okz = (lz >= -G && lz < nz + G);
      for (int idx = tid; idx < P2; idx += nt) {
        const int ex = idx % P2X, ey = idx / P2X;
        const int64_t x = tx0 - 2 + ex, y = ty0 - 2 + ey;
        double v = 0.0;
        if (okz && x >= 0 && x < m && y >= 0 && y < m) v = U[lz * pl + y * m + x];
        dst[idx] = v;
      }
    };
    // prologue: U planes zs-2, zs-1
    loadU(zs - 2);
    loadU(zs - 1);
    for (int64_t p = zs - 1; p <= ze; ++p) {
      __syncthreads();
      loadU(p + 1);
#pragma unroll
      for (int l = 0; l < KM - 1; ++l) {
        if (l < nv) {
          const double* V = cf.V[l] + a.off;
          double* dst = sV + (l * 2 + (int)(((p % 2) + 2) % 2)) * P1;
          const bool okz = (p >= -G && p < nz + G);
          for (int idx = tid; idx < P1; idx += nt) {
            const int ex = idx % P1X, ey = idx / P1X;
            const int64_t x = tx0 - 1 + ex, y = ty0 - 1 + ey;
            double v = 0.0;
            if (okz && x >= 0 && x < m && y >= 0 && y < m) v = V[p * pl + y * m + x];
            dst[idx] = v;
          }
        }
      }
      __syncthreads();
      {  // W plane p (1-halo)
        const double* u0 = sU + (int)((((p - 1) % 3) + 3) % 3) * P2;
        const double* u1 = sU + (int)(((p % 3) + 3) % 3) * P2;
        const double* u2 = sU + (int)((((p + 1) % 3) + 3) % 3) * P2;
        double* wd = sW + (int)(((p % 3) + 3) % 3) * P1;
        const int vs = (int)(((p % 2) + 2) % 2);
        const int64_t gz = z0 + p;
        const bool zin = (gz >= 0 && gz < m && p >= 1 - G && p < nz + G - 1);
        for (int idx = tid; idx < P1; idx += nt) {
          const int ex = idx % P1X, ey = idx / P1X;
          const int64_t x = tx0 - 1 + ex, y = ty0 - 1 + ey;
          double w = 0.0;
          if (zin && x >= 0 && x < m && y >= 0 && y < m) {
            const int c = (ey + 1) * P2X + ex + 1;
            const double u = u1[c];
            const double Au = cc * u + cm * (u1[c - 1] + u1[c - P2X] + u0[c]) +
                              cp * (u1[c + 1] + u1[c + P2X] + u2[c]);
            w = alpha * Au + beta_u * u;
#pragma unroll
            for (int l = 0; l < KM - 1; ++l)
              if (l < nv) w += cf.c[l] * sV[(l * 2 + vs) * P1 + idx];
          }
          wd[idx] = w;
        }
      }
      __syncthreads();
      if (p >= zs + 1) {  // consume plane c = p-1
        const int64_t cz = p - 1;
        const double* w0 = sW + (int)((((cz - 1) % 3) + 3) % 3) * P1;
        const double* w1 = sW + (int)(((cz % 3) + 3) % 3) * P1;
        const double* w2 = sW + (int)((((cz + 1) % 3) + 3) % 3) * P1;
        const double* uc = sU + (int)(((cz % 3) + 3) % 3) * P2;
        const int vs = (int)(((cz % 2) + 2) % 2);
        for (int idx = tid; idx < T3X * T3Y; idx += nt) {
          const int ex = idx % T3X, ey = idx / T3X;
          const int64_t x = tx0 + ex, y = ty0 + ey;
          if (x < m && y < m) {
            const int c = (ey + 1) * P1X + ex + 1;
            const double w = w1[c];
            const double Aw = cc * w + cm * (w1[c - 1] + w1[c - P1X] + w0[c]) +
                              cp * (w1[c + 1] + w1[c + P1X] + w2[c]);
            Wout[cz * pl + y * m + x] = w;
            acc[0] += w * w;
            acc[1] += w * Aw;
            acc[2] += Aw * Aw;
            if (cf.uslot >= 0) acc[KM + 2] += uc[(ey + 2) * P2X + ex + 2] * Aw;
#pragma unroll
            for (int l = 0; l < KM - 1; ++l)
              if (l < nv) acc[3 + l] += sV[(l * 2 + vs) * P1 + c] * Aw;
          }
        }
      }
    }
    __syncthreads();
  }
  step_epilogue<KM>(a, &cf, acc, red);
}

// ------------------------------------------------------------------------------
// y = A x (plain), and the per-column residual norms of Ritz pairs.
// ------------------------------------------------------------------------------
__global__ void apply_stencil_kernel(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off,
                                     double cc, double cm, double cp, const double* __restrict__ x,
                                     double* __restrict__ y) {
  const int64_t n = nz * plane;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
       p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = p % m;
    const int64_t q = off + p;
    const double c = x[q];
    double mn = (i > 0 ? x[q - 1] : 0.0) + x[q - m];
    double pn = (i < m - 1 ? x[q + 1] : 0.0) + x[q + m];
    if (dim == 2) {
      // y-neighbours come from ghost lines at the slab edges (zero at the boundary)
    } else {
      const int64_t jy = (p / m) % m;
      mn = (i > 0 ? x[q - 1] : 0.0) + (jy > 0 ? x[q - m] : 0.0) + x[q - plane];
      pn = (i < m - 1 ? x[q + 1] : 0.0) + (jy < m - 1 ? x[q + m] : 0.0) + x[q + plane];
    }
    y[q] = cc * c + cm * mn + cp * pn;
  }
}

// Ritz residual pieces for nvec complex vectors X = Xr + i Xi (each with ghost layout,
// pitch ld): out[v][0] += ||A x - theta x||^2, out[v][1] += ||x||^2 per block partials.
__global__ void ritz_residual_stencil_kernel(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off,
                                             int64_t ld, double cc, double cm, double cp, int nvec,
                                             const double* __restrict__ Xr, const double* __restrict__ Xi,
                                             const double* __restrict__ th_re, const double* __restrict__ th_im,
                                             double* __restrict__ partials /* [grid][nvec][2] */) {
  __shared__ double red[64];
  const int64_t n = nz * plane;
  for (int v = 0; v < nvec; ++v) {
    const double* xr = Xr + v * ld;
    const double* xi = Xi + v * ld;
    const double a = th_re[v], b = th_im[v];
    double s_res = 0.0, s_x = 0.0;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
      const int64_t i = p % m;
      const int64_t jy = (p / m) % m;
      const int64_t q = off + p;
      double ar, ai;
      {
        double mn = (i > 0 ? xr[q - 1] : 0.0), pn = (i < m - 1 ? xr[q + 1] : 0.0);
        double mi = (i > 0 ? xi[q - 1] : 0.0), pi = (i < m - 1 ? xi[q + 1] : 0.0);
        if (dim == 2) {
          mn += xr[q - m]; pn += xr[q + m]; mi += xi[q - m]; pi += xi[q + m];
        } else {
          mn += (jy > 0 ? xr[q - m] : 0.0) + xr[q - plane];
          pn += (jy < m - 1 ? xr[q + m] : 0.0) + xr[q + plane];
          mi += (jy > 0 ? xi[q - m] : 0.0) + xi[q - plane];
          pi += (jy < m - 1 ? xi[q + m] : 0.0) + xi[q + plane];
        }
        ar = cc * xr[q] + cm * mn + cp * pn;
        ai = cc * xi[q] + cm * mi + cp * pi;
      }
      // (A - theta) x, theta = a + i b:  re = ar - a xr + b xi ; im = ai - a xi - b xr
      const double rr = ar - a * xr[q] + b * xi[q];
      const double ri = ai - a * xi[q] - b * xr[q];
      s_res += rr * rr + ri * ri;
      s_x += xr[q] * xr[q] + xi[q] * xi[q];
    }
    double t[2] = {s_res, s_x};
    double o[2];
    block_sum_n<2>(t, red, o);
    if (threadIdx.x == 0) {
      partials[((int64_t)blockIdx.x * nvec + v) * 2 + 0] = o[0];
      partials[((int64_t)blockIdx.x * nvec + v) * 2 + 1] = o[1];
    }
  }
}

// ------------------------------------------------------------------------------
// host launchers
// ------------------------------------------------------------------------------
static size_t step_smem_bytes(int dim, int KM) {
  if (dim == 2) return sizeof(double) * (size_t)(E2X * E2Y + E1X * E1Y * KM);
  return sizeof(double) * (size_t)(3 * P2 + 3 * P1 + 2 * P1 * (KM - 1));
}

template <int KM>
static cudaError_t launch_step_t(const StepArgs& a, int grid, cudaStream_t st) {
  const size_t smem = step_smem_bytes(a.dim, KM);
  if (a.dim == 2) {
    if (cudaError_t e = set_smem_attr(step2d_kernel<KM>, smem)) return e;
    step2d_kernel<KM><<<grid, 256, smem, st>>>(a);
  } else {
    if (cudaError_t e = set_smem_attr(step3d_kernel<KM>, smem)) return e;
    step3d_kernel<KM><<<grid, 256, smem, st>>>(a);
  }
  return cudaGetLastError();
}

int step_km(int k) { return k <= 2 ? 2 : (k <= 4 ? 4 : 8); }

cudaError_t launch_step_stencil(const StepArgs& a, int grid, cudaStream_t st) {
  switch (step_km(a.k)) {
    case 2: return launch_step_t<2>(a, grid, st);
    case 4: return launch_step_t<4>(a, grid, st);
    default: return launch_step_t<8>(a, grid, st);
  }
}

void stencil_tiling(int dim, int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid) {
  if (dim == 2) {
    a->tiles_x = (int)((m + T2X - 1) / T2X);
    a->tiles_y = (int)((nz + T2Y - 1) / T2Y);
    a->zchunk = 0;
    a->ntiles = (int64_t)a->tiles_x * a->tiles_y;
    int64_t g = std::min<int64_t>(a->ntiles, (int64_t)num_sms * 4);
    *grid = (int)std::max<int64_t>(g, 1);
  } else {
    a->tiles_x = (int)((m + T3X - 1) / T3X);
    a->tiles_y = (int)((m + T3Y - 1) / T3Y);
    const int64_t cols = (int64_t)a->tiles_x * a->tiles_y;
    // aim for >= 3 work items per SM
    int64_t want = (int64_t)num_sms * 3;
    int64_t nch = std::max<int64_t>(1, std::min<int64_t>(nz, (want + cols - 1) / cols));
    int64_t zc = (nz + nch - 1) / nch;
    if (zc < 4) zc = std::min<int64_t>(nz, 4);
    a->zchunk = (int)zc;
    nch = (nz + zc - 1) / zc;
    a->ntiles = cols * nch;
    int64_t g = std::min<int64_t>(a->ntiles, (int64_t)num_sms * 4);
    *grid = (int)std::max<int64_t>(g, 1);
  }
}

cudaError_t launch_apply_stencil(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off, double cc,
                                 double cm, double cp, const double* x, double* y, int num_sms,
                                 cudaStream_t st) {
  int64_t n = nz * plane;
  int grid = (int)std::min<int64_t>((n + 255) / 256, (int64_t)num_sms * 8);
  if (grid < 1) grid = 1;
  apply_stencil_kernel<<<grid, 256, 0, st>>>(dim, m, nz, plane, off, cc, cm, cp, x, y);
  return cudaGetLastError();
}

cudaError_t launch_ritz_residual_stencil(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off,
                                         int64_t ld, double cc, double cm, double cp, int nvec,
                                         const double* Xr, const double* Xi, const double* thr,
                                         const double* thi, double* partials, int grid, cudaStream_t st) {
  ritz_residual_stencil_kernel<<<grid, 256, 0, st>>>(dim, m, nz, plane, off, ld, cc, cm, cp, nvec, Xr, Xi,
                                                     thr, thi, partials);
  return cudaGetLastError();
}

}  // namespace sks
