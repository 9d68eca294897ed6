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
#include <cstdio>

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

// ---- one grid barrier per column (2D, SKS_COOP1): CTA b owns the lines [z0, z1) = [b L, b L + L) of the m x nz
// grid and keeps a ring of R = k + 1 columns in shared memory, each on the lines z0-2 .. z0+L+1 (buffer line
// i <-> grid line z0-2+i).  Per column j (u = w_{j-1}, V_l the window columns):
//   fetch the two lines of u beyond the recomputed halo (z0-2, z1+1: the neighbours' own lines, from L2) with
//   cp.async, reduce the previous column's partials in step_prologue's fixed order, form w_j on lines
//   z0-1 .. z1 -- the own lines plus one recomputed halo line per side, from u and V_l already in the ring --
//   store the own lines to W, then A w_j and the next column's partial sums on the own lines; one grid barrier
//   (release/acquire counter) publishes w_j's own lines and the partials.  The halo lines computed here equal
//   the neighbours' own lines bit for bit (same operands, same operations), so w_j is the same vector as with
//   per-column launches.  The first column of a launch stages u and the window columns from W.
struct Coop1Args {
  StepArgs a;
  int j0, j1;
  int grid_prev0;
  double* part;
  int pstride;
  unsigned* sync;  // [0]: arrival counter, [1]: release flag (zero at launch); doubles at byte 64: reduced
                   // partials of the last two columns
  int lines;       // L: lines per CTA
  int ring;        // R: ring slots (k + 1)
};

__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void cp_async16_cg(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}

size_t coop1_smem(int m, int L, int ring) { return sizeof(double) * (size_t)ring * (L + 4) * m; }

// p -> (line, x) for p in [0, lines * m) without an integer division
__device__ __forceinline__ void co_split(int p, int m, float inv_m, int& li, int& x) {
  li = __float2int_rz((float)p * inv_m);
  x = p - li * m;
  if (x < 0) {
    --li;
    x += m;
  } else if (x >= m) {
    ++li;
    x -= m;
  }
}

template <int KM>
__global__ void __launch_bounds__(CO_T) step_coop1_kernel(Coop1Args ca) {
  extern __shared__ __align__(16) double co_sm[];
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ double Pr[SKS_NP];
  StepArgs a = ca.a;
  const int tid = threadIdx.x, bs = blockDim.x;
  const int m = (int)a.m, nz = (int)a.nz, L = ca.lines, R = ca.ring;
  const int BL = (L + 4) * m;  // doubles per ring slot
  const float inv_m = 1.0f / (float)m;
  const int z0 = blockIdx.x * L, z1 = min(nz, z0 + L), nl = max(0, z1 - z0);
  const double cc = a.cc, cm = a.cm, cp = a.cp;
  auto slot = [&](int c) { return co_sm + (size_t)(c % R) * BL; };
  auto colg = [&](int c, int z) { return a.W + (int64_t)c * a.ld + a.off + (int64_t)z * m; };  // grid line z
  unsigned target = 0;
#ifdef COOP1_PROF
  long long tq[6] = {0, 0, 0, 0, 0, 0}, tl = clock64();
#define CO_TICK(i)                           \
  if (tid == 0) {                         \
    const long long tn = clock64();       \
    tq[i] += tn - tl;                     \
    tl = tn;                              \
  }
#else
#define CO_TICK(i)
#endif
  for (int j = ca.j0; j <= ca.j1; ++j) {
    a.j = j;
    a.mode = 0;
    const int jm = j - 1;
    // window columns: the ones step_prologue selects (Arnoldi w_{max(0,j-k)} .. w_{j-2}, Chebyshev w_{j-2})
    const int vlo = (a.basis == 1) ? jm - 1 : max(0, j - a.k);
    const int nvs = min(KM - 1, (a.basis == 1) ? (jm >= 1 ? 1 : 0) : jm - vlo);
    double* U = slot(jm);
    // (1) staging (cp.async, before the prologue's reduction)
    if (j == ca.j0) {  // u on buffer lines 0 .. nl+3, the window columns on lines 1 .. nl+2
      const int n2 = ((nl + 4) * m) >> 1;
      const double* ug = colg(jm, z0 - 2);
      for (int p = tid; p < n2; p += bs) cp_async16_cg(U + 2 * p, ug + 2 * p);
      const int v2 = ((nl + 2) * m) >> 1;
      for (int l = 0; l < nvs; ++l) {
        const double* vg = colg(vlo + l, z0 - 1);
        double* vs = slot(vlo + l) + m;
        for (int p = tid; p < v2; p += bs) cp_async16_cg(vs + 2 * p, vg + 2 * p);
      }
    } else {  // u's lines z0-2 and z1+1 (buffer lines 0 and nl+3)
      const int h = m >> 1;
      for (int p = tid; p < 2 * h; p += bs) {
        const bool top = p >= h;
        const int q = top ? p - h : p;
        const int bl = top ? nl + 3 : 0;
        cp_async16_cg(U + bl * m + 2 * q, colg(jm, z0 - 2 + bl) + 2 * q);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    // (2) the previous column's partials (L2 loads: the ping-pong slots are rewritten every other column), in
    //     step_prologue's order: lane-strided sums (four loads in flight), then a butterfly
    double* Pg = reinterpret_cast<double*>(ca.sync + 16);  // [2][SKS_NP]
    if (j > ca.j0) {  // reduced by the last CTA to arrive at the previous column's barrier
      if (tid < SKS_NP) Pr[tid] = __ldcg(Pg + ((j - 1) & 1) * SKS_NP + tid);
      __syncthreads();
    } else {
      const double* pin = ca.part + (size_t)((j - 1) & 1) * ca.pstride * SKS_NP;
      const int gp = ca.grid_prev0;
      const int lane = tid & 31, wid = tid >> 5, nw = bs >> 5;
      for (int cmp = wid; cmp < SKS_NP; cmp += nw) {
        double t = 0.0;
        int b = lane;
        for (; b + 96 < gp; b += 128) {
          const double x0 = __ldcg(pin + (int64_t)b * SKS_NP + cmp), x1 = __ldcg(pin + (int64_t)(b + 32) * SKS_NP + cmp);
          const double x2 = __ldcg(pin + (int64_t)(b + 64) * SKS_NP + cmp),
                       x3 = __ldcg(pin + (int64_t)(b + 96) * SKS_NP + cmp);
          t += x0;
          t += x1;
          t += x2;
          t += x3;
        }
        for (; b < gp; b += 32) t += __ldcg(pin + (int64_t)b * SKS_NP + cmp);
        t = warp_sum(t);
        if (lane == 0) Pr[cmp] = t;
      }
      __syncthreads();
    }
    CO_TICK(0)
    a.partials_in = Pr;  // one pre-reduced row (exact: the prologue adds zeros to it)
    a.grid_prev = 1;
    a.partials_out = ca.part + (size_t)(j & 1) * ca.pstride * SKS_NP;
    const bool go = step_prologue(a, &cf, red);  // breakdown / early exit: the same decision in every CTA
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    if (!go) return;
    __syncthreads();
    CO_TICK(1)
    const int nv = min(cf.nv, nvs);
    const double al = cf.alpha, be = cf.beta_u;
    double* Wj = a.W + (int64_t)j * a.ld + a.off;
    double* Bj = slot(j);
    const double* Vs[KM > 1 ? KM - 1 : 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) Vs[l] = slot(vlo + (l < nvs ? l : 0));
    // (3) w_j on lines z0-1 .. z1 (buffer lines 1 .. nl+2; lines outside [0, nz) are zero)
    for (int p = m + tid; p < (nl + 3) * m; p += bs) {
      int bl, x;
      co_split(p, m, inv_m, bl, x);
      const int z = z0 - 2 + bl;
      double w = 0.0;
      if (z >= 0 && z < nz) {
        const double* u = U + p;
        const double au = cc * u[0] + cm * (u[-m] + (x > 0 ? u[-1] : 0.0)) + cp * (u[m] + (x < m - 1 ? u[1] : 0.0));
        w = fma(al, au, be * u[0]);
#pragma unroll
        for (int l = 0; l < KM - 1; ++l)
          if (l < nv) w = fma(cf.c[l], Vs[l][p], w);
        if (bl >= 2 && bl <= nl + 1) Wj[(int64_t)z * m + x] = w;
      }
      Bj[p] = w;
    }
    __syncthreads();
    CO_TICK(2)
    // (4) A w_j and the next column's partial sums on the own lines (buffer lines 2 .. nl+1)
    double acc[KM + 3];
#pragma unroll
    for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;
    for (int p = 2 * m + tid; p < (nl + 2) * m; p += bs) {
      int bl, x;
      co_split(p, m, inv_m, bl, x);
      const double* w = Bj + p;
      const double wv = w[0];
      const double aw = cc * wv + cm * (w[-m] + (x > 0 ? w[-1] : 0.0)) + cp * (w[m] + (x < m - 1 ? w[1] : 0.0));
      acc[0] = fma(wv, wv, acc[0]);
      acc[1] = fma(wv, aw, acc[1]);
      acc[2] = fma(aw, aw, acc[2]);
#pragma unroll
      for (int l = 0; l < KM - 1; ++l)
        if (l < nv && cf.vslot[l] >= 0) acc[3 + l] = fma(Vs[l][p], aw, acc[3 + l]);
      if (cf.uslot >= 0) acc[KM + 2] = fma(U[p], aw, acc[KM + 2]);
    }
    step_epilogue<KM>(a, &cf, acc, red);
    // (5) grid barrier: publish w_j's own lines and the partials.  The last CTA to arrive reduces the partials
    //     (step_prologue's fixed order) into Pg[j & 1] before releasing the others: one CTA reads the grid's rows
    //     instead of every CTA (the all-to-all read of the same few kB serialises in the L2 slices)
    target += gridDim.x;
    __syncthreads();
    CO_TICK(3)
    __shared__ int co_last;
    if (tid == 0) {
      __threadfence();
      co_last = (atomicAdd(ca.sync, 1u) == target - 1);
      __threadfence();
    }
    __syncthreads();
    if (co_last) {
      if (j < ca.j1) {
        const double* pin = a.partials_out;
        const int gp = (int)gridDim.x;
        const int lane = tid & 31, wid = tid >> 5, nw = bs >> 5;
        for (int cmp = wid; cmp < SKS_NP; cmp += nw) {
          double t = 0.0;
          int b = lane;
          for (; b + 96 < gp; b += 128) {
            const double x0 = __ldcg(pin + (int64_t)b * SKS_NP + cmp),
                         x1 = __ldcg(pin + (int64_t)(b + 32) * SKS_NP + cmp);
            const double x2 = __ldcg(pin + (int64_t)(b + 64) * SKS_NP + cmp),
                         x3 = __ldcg(pin + (int64_t)(b + 96) * SKS_NP + cmp);
            t += x0;
            t += x1;
            t += x2;
            t += x3;
          }
          for (; b < gp; b += 32) t += __ldcg(pin + (int64_t)b * SKS_NP + cmp);
          t = warp_sum(t);
          if (lane == 0) __stcg(Pg + (j & 1) * SKS_NP + cmp, t);
        }
        __syncthreads();
      }
      if (tid == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ca.sync + 1), "r"((unsigned)(j - ca.j0 + 1))
                     : "memory");
      }
    } else if (tid == 0) {
      while (ld_acquire_u32(ca.sync + 1) < (unsigned)(j - ca.j0 + 1)) __nanosleep(20);
    }
    __syncthreads();
    CO_TICK(4)
  }
#ifdef COOP1_PROF
  if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1))
    printf("coop1 cta %d cols %d: reduce %lld prologue %lld w %lld Aw+epi %lld barrier %lld cycles/col\n", blockIdx.x,
           ca.j1 - ca.j0 + 1, tq[0] / (ca.j1 - ca.j0 + 1), tq[1] / (ca.j1 - ca.j0 + 1), tq[2] / (ca.j1 - ca.j0 + 1),
           tq[3] / (ca.j1 - ca.j0 + 1), tq[4] / (ca.j1 - ca.j0 + 1));
#endif
#undef CO_TICK
}

int coop_grid(int main_sms) {
  int per = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, step_coop_kernel<4>, CO_T, 0) != cudaSuccess || per < 1) {
    cudaGetLastError();
    return 0;
  }
  return main_sms * std::min(per, 1);
}

// lines per CTA of the one-barrier kernel (2D, m even; 0 = not applicable): at least ~2048 points per CTA, at most
// `max_grid` CTAs, shared memory within the opt-in limit
int coop1_lines(int dim, int64_t m, int64_t nz, int k, int max_grid) {
  if (dim != 2 || (m & 1) || max_grid < 1 || nz < 2) return 0;
  int L = (int)std::max<int64_t>((nz + max_grid - 1) / max_grid, (2048 + m - 1) / m);
  L = (int)std::min<int64_t>(L, nz);
  if (coop1_smem((int)m, L, std::max(k + 1, 3)) > 220 * 1024) return 0;
  return L;
}

cudaError_t launch_step_coop1(const StepArgs& a, int j0, int j1, int grid_prev0, double* part, int pstride,
                              unsigned* sync, int lines, cudaStream_t st) {
  Coop1Args ca;
  ca.a = a;
  ca.j0 = j0;
  ca.j1 = j1;
  ca.grid_prev0 = grid_prev0;
  ca.part = part;
  ca.pstride = pstride;
  ca.sync = sync;
  ca.lines = lines;
  ca.ring = std::max(a.k + 1, 3);  // Chebyshev: u = w_{j-1}, V = w_{j-2}, w_j
  const int grid = (int)((a.nz + lines - 1) / lines);
  cudaError_t e = cudaMemsetAsync(sync, 0, 2 * sizeof(unsigned), st);
  if (e != cudaSuccess) return e;
  void* args[] = {&ca};
  const void* fn;
  const int km = step_km(a.k);
  switch (km) {
    case 2: fn = (const void*)step_coop1_kernel<2>; break;
    case 4: fn = (const void*)step_coop1_kernel<4>; break;
    default: fn = (const void*)step_coop1_kernel<8>; break;
  }
  const size_t smem = coop1_smem((int)a.m, lines, ca.ring);
  e = set_smem_attr_raw(fn, smem);
  if (e != cudaSuccess) return e;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(CO_T), args, smem, st);
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
