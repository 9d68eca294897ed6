// step.cuh -- argument block and coefficient prologue of the fused Arnoldi step.
//
// One launch produces one new (unnormalised) basis column w_j of the k-truncated
// Arnoldi recurrence (Eq. partorth; Alg. 1):
//     w_j = m_{j-1} - sum_{i=j-k}^{j-1} h_i b_i,   h_i = <b_i, m_{j-1}>,  m_{j-1} = A b_{j-1}
// with b_i = sigma_i w_i (sigma_i = 1/||w_i||, reading O9: columns stored unnormalised).
// m_{j-1} is recomputed on the fly from w_{j-1} (matrix-free A), and in the SAME pass
// the kernel forms A w_j and the partial sums the NEXT step needs:
//     ||w_j||^2, <w_j, A w_j>, ||A w_j||^2, <w_i, A w_j> (i = j-k+1..j-1)
// so h^{(j+1)} = { sigma_j sigma_i <w_i, A w_j>,  sigma_j^2 <w_j, A w_j> } are known at
// the start of launch j+1 without another pass over memory.  Each CTA of launch j+1
// re-reduces the per-CTA partials of launch j in a fixed order (deterministic).
#pragma once
#include "common.cuh"

struct StepArgs {
  // geometry (stencil): local slab of nz planes (2D: lines) starting at global plane z0
  int64_t m;        // points per side
  int64_t nz;       // local planes
  int64_t z0;       // global index of the first local plane
  int64_t plane;    // points per plane (m or m*m)
  int64_t ld;       // column pitch (doubles)
  int64_t off;      // offset of the first interior point (= G*plane)
  int G;            // ghost planes per side
  int dim;
  double cc, cm, cp;  // stencil coefficients: centre, minus-neighbours, plus-neighbours
  // recurrence
  int mode;         // 0: step j >= 1;  1: w_0 = f - A x;  2: w_0 = v0
  int j, k;
  double* W;        // column i at W + i*ld
  const double* xin;  // mode 1: x;   mode 2: v0
  const double* fin;  // mode 1: f
  const double* partials_in;  // [grid_prev][SKS_NP] of launch j-1
  int grid_prev;
  double* partials_out;       // [gridDim.x][SKS_NP]
  double* sigma;    // sigma_i = 1/||w_i||
  double* H;        // Hbar, column-major, ld = ldH: Hbar[i, j] = h coefficient of b_i in w_{j+1}
  int ldH;
  double* mnorm;    // ||m_i||
  double* gam;      // gam_i: A b_i = gam_i w_{i+1} + sum_l H[l, i] b_l  (1 for Arnoldi)
  int basis;        // 0: k-truncated Arnoldi (Eq. partorth), 1: Chebyshev (Eq. Chebrecurse)
  double cheb_c, cheb_rho, cheb_e;  // Chebyshev: centre, rho, (dx^2 - dy^2)/(4 rho)
  int defer;        // Chebyshev: from column 2 on the recurrence coefficients are constants, so
                    // launches j >= 3 skip the previous launch's partials; the norms, sigma and the recurrence
                    // bookkeeping of a whole batch are finalised at once (cheb_finalize_kernel)
  int fe;           // forward-edge step (3D z-march, k <= 2; set by the launcher): the kernel produces
                    // ||w||^2, <w,Aw> = cc ||w||^2 + (cm+cp) sum_{forward edges} w_p w_q and <U,Aw> = <A^T U,w>
                    // but not ||A w||^2, so the breakdown reference ||m_{j-1}|| is derived (reading O39)
  CtrlBlock* ctrl;
  int64_t ntiles;   // work items
  int tiles_x, tiles_y, zchunk;  // tiling
};

struct StepCoef {
  const double* U;  // vector whose A-image is taken (w_{j-1}, x, or v0)
  double alpha;     // coefficient of A U
  double beta_u;    // coefficient of U itself
  int nv;           // number of extra vectors
  const double* V[SKS_KMAX];
  double c[SKS_KMAX];
  int vslot[SKS_KMAX];  // output partial slot of <V_l, A w>, -1 = none
  int uslot;            // output partial slot of <U, A w>, -1 = none
  int ok;
};

// Computes the coefficients of this launch into smem `cf` (block-uniform). Returns false
// (for the whole block) if the basis has stopped (breakdown) -> nothing to do.
__device__ __forceinline__ bool step_prologue(const StepArgs& a, StepCoef* cf, double* red) {
  const int tid = threadIdx.x;
  if (a.mode != 0) {
    if (tid == 0) {
      cf->ok = 1;
      cf->U = a.xin;
      cf->alpha = (a.mode == 1) ? -1.0 : 0.0;
      cf->beta_u = (a.mode == 2) ? 1.0 : 0.0;
      cf->nv = (a.mode == 1) ? 1 : 0;
      cf->V[0] = a.fin;
      cf->c[0] = 1.0;
      cf->vslot[0] = -1;
      cf->uslot = -1;
    }
    __syncthreads();
    return true;
  }
  if (a.defer && a.basis == 1 && a.j >= 3) {
    // deferred Chebyshev step: w_j = [(A - cI) w_{j-1} - e w_{j-2}] / rho on the raw vectors (Eq. Chebrecurse
    // P:1192-1199), no dependence on the norms -- no reduction, no grid-wide synchronisation per column
    if (tid == 0) {
      const int jm = a.j - 1;
      cf->ok = (a.ctrl->stop_col > jm && a.ctrl->exit_cols == 0) ? 1 : 0;
      const double rho = a.cheb_rho;
      cf->U = a.W + (int64_t)jm * a.ld;
      cf->alpha = 1.0 / rho;
      cf->beta_u = -a.cheb_c / rho;
      cf->nv = 1;
      cf->V[0] = a.W + (int64_t)(jm - 1) * a.ld;
      cf->c[0] = -a.cheb_e / rho;
      cf->vslot[0] = -1;
      cf->uslot = -1;
    }
    __syncthreads();
    return cf->ok != 0;
  }
  // fixed-order reduction of the previous launch's partials: warp w sums component w (w + nwarps, ...) over the
  // grid_prev rows (lane-strided, then a butterfly) -- one barrier, ~5 shuffles per component, instead of a
  // block-wide reduction of all SKS_NP components by every thread
  // Only components 0 .. k+1 are read below (the window dots end at slot k+1).  Each lane issues all of its loads
  // before the first add (the partials were written by the previous launch and sit in L2: a load-add loop would be a
  // chain of L2 round trips); the sums keep the lane-strided sequential order.
  __shared__ double P[SKS_NP];
  // thread 0's scalar state (stop/exit flags, sigma, ||m||, gamma, the H column of the FE breakdown reference) is
  // loaded before the reduction, so its latency overlaps the partials' instead of following the barrier
  const int j = a.j, k = a.k;
  const int jm = j - 1;
  const int lo = max(0, j - k);
  int stop_col = 0, exit_cols = 0;
  double sgw[SKS_KMAX], hcw[SKS_KMAX], s_jm1 = 1.0, s_0 = 1.0, mn_jm1 = 0.0, gm_jm1 = 0.0;
  if (tid == 0) {
    stop_col = a.ctrl->stop_col;
    exit_cols = a.ctrl->exit_cols;
#pragma unroll
    for (int l = 0; l < SKS_KMAX; ++l) sgw[l] = (lo + l <= jm - 1) ? a.sigma[lo + l] : 0.0;
    const int lo2 = max(0, jm - k);
#pragma unroll
    for (int l = 0; l < SKS_KMAX; ++l)
      hcw[l] = (a.fe && jm >= 1 && lo2 + l <= jm - 1) ? a.H[(lo2 + l) + (int64_t)(jm - 1) * a.ldH] : 0.0;
    if (jm >= 1) {
      s_jm1 = a.sigma[jm - 1];
      mn_jm1 = a.mnorm[jm - 1];
      gm_jm1 = a.gam[jm - 1];
    }
    s_0 = a.sigma[0];
  }
  {
    const int lane = tid & 31, wid = tid >> 5, nw = (int)(blockDim.x >> 5);
    const int ncmp = min(SKS_NP, k + 2);
    for (int cmp = wid; cmp < ncmp; cmp += nw) {
      double t = 0.0;
      for (int b0 = lane; b0 < a.grid_prev; b0 += 256) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + 32 * u;
          v[u] = (b < a.grid_prev) ? a.partials_in[(int64_t)b * SKS_NP + cmp] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) t += v[u];
      }
      t = warp_sum(t);
      if (lane == 0) P[cmp] = t;
    }
    if (tid >= ncmp && tid < SKS_NP) P[tid] = 0.0;
    __syncthreads();
  }
  (void)red;
  if (tid == 0) {
    cf->ok = 1;
    if (stop_col <= jm || exit_cols != 0) cf->ok = 0;
    const double N = P[0];
    const double nu = sqrt(N);
    bool bd = !(N > 0.0) || !isfinite(N);
    // breakdown (reading O10): ||w_j|| negligible against the scale of the vector it came from
    // (Arnoldi: ||A b_{j-1}||; Chebyshev: the previous raw vector, raw_0 = b_0 has norm 1)
    double ref = (a.basis == 1) ? (jm >= 2 ? 1.0 / s_jm1 : 1.0) : (jm >= 1 ? mn_jm1 : 0.0);
    if (a.basis == 0 && jm >= 1 && ref < 0.0) {
      // forward-edge launches leave ||m_{jm-1}|| as the marker -1: m_{jm-1} = A b_{jm-1} = w_jm + sum_l H[l, jm-1] b_l
      // over a window of k+1 consecutive columns, which k-truncated Arnoldi makes orthonormal (Eq. partorth
      // P:208-218), so ||m_{jm-1}||^2 = ||w_jm||^2 + sum_l H[l, jm-1]^2 (reading O39)
      double s2 = N;
#pragma unroll
      for (int l = 0; l < SKS_KMAX; ++l) s2 += hcw[l] * hcw[l];  // zero beyond the window
      ref = sqrt(s2);
    }
    if (jm >= 1 && nu <= 1e-14 * ref) bd = true;
    if (cf->ok && bd) {
      cf->ok = 0;
      if (blockIdx.x == 0) {
        a.ctrl->stop_col = jm;
        a.ctrl->breakdown = 1;
        if (jm >= 1) a.H[jm + (int64_t)(jm - 1) * a.ldH] = gm_jm1 * nu;
        if (jm == 0) a.ctrl->rnorm = nu;
      }
    }
    if (cf->ok) {
      const double sg = 1.0 / nu;
      cf->U = a.W + (int64_t)jm * a.ld;
      if (a.basis == 1) {
        // Chebyshev on the raw vectors w: w_1 = (A - cI) b_0 / (2 rho) with
        // b_0 = sg w_0; w_j = [(A - cI) w_{j-1} - e raw_{j-2}] / rho, raw_0 = b_0 = sigma_0 w_0
        const double rho = a.cheb_rho, cc0 = a.cheb_c, e = a.cheb_e;
        const double s0 = (jm == 0) ? sg : 1.0;  // only the first vector is used normalised
        const double al = (jm == 0) ? s0 / (2.0 * rho) : 1.0 / rho;
        cf->alpha = al;
        cf->beta_u = -cc0 * al;
        cf->nv = (jm >= 1) ? 1 : 0;
        if (jm >= 1) {
          cf->V[0] = a.W + (int64_t)(jm - 1) * a.ld;
          cf->c[0] = -(e / rho) * (jm == 1 ? s_0 : 1.0);
          cf->vslot[0] = -1;
        }
      } else {
        const double hj = sg * sg * P[1];
        cf->alpha = sg;
        cf->beta_u = -hj * sg;
        const int nv = jm - lo;
        cf->nv = nv;
#pragma unroll
        for (int l = 0; l < SKS_KMAX; ++l) {
          if (l >= nv) break;
          const int i = lo + l;
          const double si = sgw[l];
          const double hi = sg * si * P[3 + i - (j - k)];
          cf->V[l] = a.W + (int64_t)i * a.ld;
          cf->c[l] = -hi * si;
          const int sl = i - (j - k + 1);
          cf->vslot[l] = (sl >= 0) ? 3 + sl : -1;
        }
      }
      cf->uslot = (a.basis == 0 && k >= 2) ? k + 1 : -1;
      if (blockIdx.x == 0) {
        // recurrence of column jm (both bases): A b_jm = gam w_j + sum_l H[l, jm] b_l with
        // gam = sg/alpha, H[jm, jm] = -beta_u/alpha, H[i, jm] = -sg c_i / (alpha sigma_i)
        const double al = cf->alpha;
        const double gm = sg / al;
        a.gam[jm] = gm;
        a.H[jm + (int64_t)jm * a.ldH] = -cf->beta_u / al;
        const int nvb = cf->nv;
#pragma unroll
        for (int l = 0; l < SKS_KMAX; ++l) {
          if (l >= nvb) break;
          const int i = (a.basis == 1) ? jm - 1 : lo + l;
          const double si = (a.basis == 1) ? s_jm1 : sgw[l];
          a.H[i + (int64_t)jm * a.ldH] = -sg * cf->c[l] / (al * si);
        }
        a.sigma[jm] = sg;
        a.mnorm[jm] = a.fe ? -1.0 : sg * sqrt(P[2]);
        if (jm >= 1) a.H[jm + (int64_t)(jm - 1) * a.ldH] = gm_jm1 * nu;
        if (jm == 0) a.ctrl->rnorm = nu;
      }
    }
  }
  __syncthreads();
  return cf->ok != 0;
}

// write the block's partials into the output slots
template <int KM>
__device__ __forceinline__ void step_epilogue(const StepArgs& a, const StepCoef* cf,
                                              double (&acc)[KM + 3], double* red) {
  // per-warp butterflies, then warp v finishes value v over the warps (fixed order) and the block's
  // SKS_NP partial slots are written from shared memory (two barriers; no serial pass over all values)
  __shared__ double R[SKS_NP];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = warp_sum(acc[i]);
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < KM + 3; ++i) red[i * 32 + wid] = acc[i];
  }
  if (threadIdx.x < SKS_NP) R[threadIdx.x] = 0.0;
  __syncthreads();
  for (int v = wid; v < KM + 3; v += nw) {
    double t = lane < nw ? red[v * 32 + lane] : 0.0;
    t = warp_sum(t);
    if (lane == 0) {
      int slot = -1;
      if (v < 3) slot = v;
      else if (v < KM + 2) slot = (v - 3 < cf->nv) ? cf->vslot[v - 3] : -1;
      else slot = cf->uslot;
      if (slot >= 0) R[slot] = t;
    }
  }
  __syncthreads();
  if (threadIdx.x < SKS_NP) a.partials_out[(int64_t)blockIdx.x * SKS_NP + threadIdx.x] = R[threadIdx.x];
}
