// stencil_zm.cu -- fused truncated-Arnoldi step for the 3D 7-point operator, z-march design.
//
// Same arithmetic as step.cuh / stencil.cu (one launch produces w_j and the next step's
// partial sums, Eq. partorth, Alg. 1), organised to minimise on-chip
// traffic:
//
//   * a CTA owns an xy tile of TX x TY = 32 x 16 output columns and marches through a range
//     of z planes, ZS planes per step; all CTAs together get equal shares of the
//     (tile, plane) units, so the persistent grid (one CTA per SM) is balanced for any m
//     and slab depth;
//   * per step the TMA brings ZS+2 U planes (36 x 20, 2-point xy halo) and ZS planes of each
//     window vector V_l (36 x 18) into one of two stages (mbarrier completion; the next
//     step's stage is in flight during this step); out-of-bounds boxes are zero-filled, so
//     the Dirichlet x/y boundary costs nothing;
//   * each of the 34 x 18 W-box threads owns one xy column: it forms w_j for ZS planes from
//     the staged U/V (z neighbours in registers), stores them into a ring of 2 ZS + 2 w_j
//     planes, and -- after ONE __syncthreads per step -- interior threads form A w_j for
//     the ZS planes one behind, store w_j and accumulate ||w||^2, <w,Aw>, ||Aw||^2 and the
//     window dots in registers.
#include <cudaTypedefs.h>

#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "step.cuh"
#include "tma.cuh"

namespace sks {

#ifndef ZM_TX
#define ZM_TX 32
#endif
#ifndef ZM_TY
#define ZM_TY 16
#endif
#ifndef ZM_CPS
#define ZM_CPS 1  // resident CTAs per SM
#endif
constexpr int ZX = ZM_TX, ZY = ZM_TY;            // output tile
constexpr int ZWX = ZX + 2, ZWY = ZY + 2;        // W box 34 x 18 (one thread per column)
constexpr int ZUX = ZX + 4, ZUY = ZY + 4;        // U plane box 36 x 20
constexpr int ZVX = ZX + 4, ZVY = ZY + 2;        // V plane box 36 x 18 (origin x0-2: 16-byte aligned)
constexpr int ZUP = ZUX * ZUY;                   // 720 doubles per U plane
constexpr int ZVP = ZVX * ZVY;                   // 648 doubles per V plane
constexpr int ZW = ZWX * ZWY;                    // 612
#ifndef ZM_PITCH
#define ZM_PITCH 0
#endif
// ZM_PITCH=1: thread rows and w_j ring rows use the U-plane pitch (36), so every warp touches one
// contiguous run of shared memory per load (no row-break bank conflicts; 2 idle threads per row).
// Measured 38.8 us vs 38.1 us at C3 (the conflicts are not the bound), so off by default.
constexpr int ZRX = ZM_PITCH ? ZUX : ZWX;        // thread-row width = ring row pitch
constexpr int ZR = ZRX * ZWY;                    // ring plane (648 doubles)
constexpr int ZT = (ZRX * ZWY + 31) / 32 * 32;
#ifndef ZM_BALANCE_DEFAULT
#define ZM_BALANCE_DEFAULT 1
#endif
#ifndef ZM_NEXT
#define ZM_NEXT 1  // pair kernel: prefetch the next piece's first stages during this piece's last steps
#endif
#ifndef ZM_EARLY
#define ZM_EARLY 1  // pair kernel: issue the first two stages before the prologue's reduction
#endif
#ifndef ZM_NPY_DEFAULT
#define ZM_NPY_DEFAULT 2
#endif  // threads (32 x 16 tile: 672 = 21 warps)

constexpr int ZM_MAXG = 2 * 148;  // CTAs covered by the partition table
struct ZmArgs {
  int ucol;
  int vcol[SKS_KMAX];
  int ncolxy;      // xy tiles
  int tiles_x;
  int64_t units;   // ncolxy * nz
  int nv;          // window vectors of this launch (= StepCoef::nv, known on the host)
  int vdot;        // bit l: the dot <V_l, A w_j> is needed by the next step (its partial slot is used)
  int store_b;     // warp-specialised kernel: w_j is stored by group B (1) or group A (0)
  int use_ub;      // 1: CTA b owns units [ub[b], ub[b+1]) (step-balanced partition), else proportional
  int32_t ub[ZM_MAXG + 1];
};

__host__ __device__ constexpr int zm_al16(int d) { return (d + 15) & ~15; }  // 128-byte multiple (doubles)
template <int KM, int ZS>
__host__ __device__ constexpr int zm_ublk() { return zm_al16(ZUP * (ZS + 2)); }
template <int KM, int ZS>
__host__ __device__ constexpr int zm_vblk() { return zm_al16(ZVP * ZS); }
template <int KM, int ZS>
__host__ __device__ constexpr int zm_stage() { return zm_ublk<KM, ZS>() + (KM - 1) * zm_vblk<KM, ZS>(); }
template <int KM, int ZS, int NSTG>
__host__ __device__ constexpr size_t zm_smem_bytes_n() {
  return 128 + sizeof(double) * ((size_t)NSTG * zm_stage<KM, ZS>() + (size_t)(3 * ZS) * ZR);
}
template <int KM, int ZS>
__host__ __device__ constexpr size_t zm_smem_bytes() {
  return 128 + sizeof(double) * ((size_t)2 * zm_stage<KM, ZS>() + (size_t)(3 * ZS) * ZR);
}

template <int KM, int ZS, bool FULL, bool USL>
__global__ void __launch_bounds__(ZT, ZM_CPS)
    step3d_zm_kernel(StepArgs a, ZmArgs z, const __grid_constant__ CUtensorMap tmU,
                     const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smraw_z[];
  double* sm = reinterpret_cast<double*>(smraw_z + ((128u - (smem_u32(smraw_z) & 127u)) & 127u));
  constexpr int STG = zm_stage<KM, ZS>();
  constexpr int UB = zm_ublk<KM, ZS>(), VB = zm_vblk<KM, ZS>();
  constexpr int R = 3 * ZS;  // w_j plane ring: plane p in slot (p - wa + ZS) mod 3 ZS
  double* ring = sm + 2 * STG;
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  // PDL: everything above overlaps the previous kernel's tail; its outputs (partials, w_{j-1}) are
  // read only after this wait.  The next step launch may be scheduled as soon as this grid runs.
  pdl_wait_and_release();
  if (!step_prologue(a, &cf, red)) return;  // contains __syncthreads
  const int nv = FULL ? KM - 1 : cf.nv;
  const uint32_t sbytes = (uint32_t)(ZUP * (ZS + 2) * 8 + nv * ZVP * ZS * 8);
  const int m = (int)a.m, nz = (int)a.nz, z0g = (int)a.z0, G = a.G;
  const int64_t pl = a.plane;
  const double cc = a.cc, cm = a.cm, cp = a.cp, alpha = cf.alpha, beta_u = cf.beta_u;
  double cl[KM - 1];
#pragma unroll
  for (int l = 0; l < KM - 1; ++l) cl[l] = (l < nv) ? cf.c[l] : 0.0;
  constexpr bool uslot = USL;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;

  // this thread's W-box column
  // threads past the last thread row shadow the last W column (no stores); threads in the pitch
  // padding of a row (bx >= ZWX) compute in-bounds garbage and store nothing
  const int tcol = tid < ZR ? tid : ZR - ZRX + ZWX - 1;
  const int bx = tcol % ZRX, by = tcol / ZRX;
  const bool wt = tid < ZR && bx < ZWX;
  const int cu = (by + 1) * ZUX + (bx + 1);  // U-plane offset of the column
  const int cvv = by * ZVX + (bx + 1);       // V-plane offset
  const int cwb = by * ZRX + bx;             // ring-plane offset
  const bool inner = wt && bx >= 1 && bx <= ZX && by >= 1 && by <= ZY;

  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;

  uint32_t phase = 0;  // parity bits of the two stage barriers
  uint32_t sidx = 0;   // global stage counter (slot = sidx & 1)
  const int64_t u_lo = z.use_ub ? (int64_t)z.ub[blockIdx.x] : (z.units * blockIdx.x) / gridDim.x;
  const int64_t u_hi = z.use_ub ? (int64_t)z.ub[blockIdx.x + 1] : (z.units * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t u = u_lo; u < u_hi;) {
    const int col = (int)(u / nz);
    const int za = (int)(u % nz);
    const int64_t zr = za + (u_hi - u);
    const int zb = (int)(zr < nz ? zr : nz);
    u += zb - za;
    const int tx = col % z.tiles_x, ty = col / z.tiles_x;
    const int x0 = tx * ZX, y0 = ty * ZY;
    const int wa = za - 1;                         // first w_j plane of the piece
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;  // w_j planes wa .. zb
    const uint32_t s0 = sidx;
    auto issue = [&](int t) {  // stage t: U planes [wa+t ZS-1, wa+t ZS+ZS], V planes [wa+t ZS, +ZS)
      const uint32_t slot = (s0 + (uint32_t)t) & 1u;
      double* dst = sm + slot * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[slot], sbytes);
      tma_load_4d(dst, &tmU, &bar[slot], x0 - 2, y0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB + l * VB, &tmV, &bar[slot], x0 - 2, y0 - 1, p0 + G, z.vcol[l]);
    };
    if (tid == 0) {
      issue(0);
      if (nsteps > 1) issue(1);
    }
    double wp1 = 0.0, wp2 = 0.0;  // w_j at planes p0-1, p0-2 (carried)
    double vlast[KM - 1];         // V_l at plane p0-1 (carried)
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) vlast[l] = 0.0;
    const int gxw = x0 - 1 + bx, gyw = y0 - 1 + by;  // global xy of this W column
    const bool xyin = wt && (unsigned)gxw < (unsigned)m && (unsigned)gyw < (unsigned)m;
    const bool aw = inner && gxw < m && gyw < m;    // this thread forms A w_j (interior output)
    double* wcol = Wout + (int64_t)(wa - 1) * pl + (int64_t)gyw * m + gxw;  // plane wa-1 of the column
    // Fast steps (CTA-uniform: every plane of the step inside the piece and the domain, t >= T0)
    // run without per-plane predicates; the xy mask is folded into the coefficients (a column
    // outside the domain gets w = 0 A u + 0 u + 0 v = 0).  The w_j ring has period 3 steps, so
    // the step body is instantiated for the 3 ring phases and every ring offset is a constant.
    const double am = xyin ? alpha : 0.0, bm = xyin ? beta_u : 0.0;
    double clm[KM - 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) clm[l] = xyin ? cl[l] : 0.0;
    constexpr int T0 = ZS == 1 ? 2 : 1;
    auto step = [&](int t, auto phc) {
      constexpr int PH = decltype(phc)::value;
      constexpr int SBW = ((PH + 1) % 3) * ZS;          // ring slot of plane p0
      constexpr int SBP = SBW == 0 ? R - 1 : SBW - 1;   // ring slot of plane p0-1
      const uint32_t slot = (s0 + (uint32_t)t) & 1u;
      mbar_wait(&bar[slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
      const double* sU = sm + slot * STG;
      const double* sV = sU + UB;
      const int p0 = wa + t * ZS;
      const bool fast = t >= T0 && p0 + ZS - 1 <= zb && z0g + p0 + ZS - 1 < m;
      double w[ZS], c[ZS + 2], v[KM - 1][ZS];
      double* rw = ring + SBW * ZR + cwb;        // plane p0 (+ i ZR for p0 + i)
      const double* rp = ring + SBP * ZR + cwb;  // plane p0-1
      // ---- w_j on planes p0 .. p0+ZS-1 (this thread's column)
#pragma unroll
      for (int k = 0; k < ZS + 2; ++k) c[k] = sU[k * ZUP + cu];
      if (fast) {
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
#pragma unroll
          for (int l = 0; l < KM - 1; ++l) v[l][i] = (FULL || l < nv) ? sV[l * VB + i * ZVP + cvv] : 0.0;
          const double* q = sU + (i + 1) * ZUP + cu;
          const double Au = cc * c[i + 1] + cm * (q[-1] + q[-ZUX] + c[i]) + cp * (q[1] + q[ZUX] + c[i + 2]);
          double wv = am * Au + bm * c[i + 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (FULL || l < nv) wv += clm[l] * v[l][i];
          w[i] = wv;
          if (wt) rw[i * ZR] = wv;
        }
      } else {
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
          const int p = p0 + i;
#pragma unroll
          for (int l = 0; l < KM - 1; ++l) v[l][i] = (FULL || l < nv) ? sV[l * VB + i * ZVP + cvv] : 0.0;
          const double* q = sU + (i + 1) * ZUP + cu;
          const double Au = cc * c[i + 1] + cm * (q[-1] + q[-ZUX] + c[i]) + cp * (q[1] + q[ZUX] + c[i + 2]);
          double wv = alpha * Au + beta_u * c[i + 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (FULL || l < nv) wv += cl[l] * v[l][i];
          wv = (xyin && (unsigned)(z0g + p) < (unsigned)m && p <= zb) ? wv : 0.0;
          w[i] = wv;
          if (wt) rw[i * ZR] = wv;
        }
      }
      __syncthreads();
      if (tid == 0 && t + 2 < nsteps) issue(t + 2);  // the stage just consumed is free
      // ---- A w_j on planes p0-1 .. p0+ZS-2
      if (aw) {
        double* wo = wcol;
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
          const int qp = p0 - 1 + i;
          if (fast || (qp >= za && qp < zb)) {
            const double wq = (i == 0) ? wp1 : w[i - 1];
            const double wqm = (i == 0) ? wp2 : (i == 1 ? wp1 : w[i - 2]);
            const double* r = (i == 0) ? rp : rw + (i - 1) * ZR;
            const double Aw = cc * wq + cm * (r[-1] + r[-ZRX] + wqm) + cp * (r[1] + r[ZRX] + w[i]);
            *wo = wq;
            acc[0] += wq * wq;
            acc[1] += wq * Aw;
            acc[2] += Aw * Aw;
            if (uslot) acc[KM + 2] += c[i] * Aw;
#pragma unroll
            for (int l = 0; l < KM - 1; ++l)
              if (FULL || l < nv) acc[3 + l] += ((i == 0) ? vlast[l] : v[l][i - 1]) * Aw;
          }
          wo += pl;
        }
      }
      if (ZS >= 2) {
        wp2 = w[ZS >= 2 ? ZS - 2 : 0];
        wp1 = w[ZS - 1];
      } else {
        wp2 = wp1;
        wp1 = w[0];
      }
#pragma unroll
      for (int l = 0; l < KM - 1; ++l) vlast[l] = v[l][ZS - 1];
      wcol += (int64_t)ZS * pl;
    };
    for (int t = 0; t < nsteps; t += 3) {
      step(t, std::integral_constant<int, 0>{});
      if (t + 1 < nsteps) step(t + 1, std::integral_constant<int, 1>{});
      if (t + 2 < nsteps) step(t + 2, std::integral_constant<int, 2>{});
    }
    sidx = s0 + (uint32_t)nsteps;
    __syncthreads();  // ring and stages are reused by the next piece
  }
  step_epilogue<KM>(a, &cf, acc, red);
}

// ---- paired-column variant (default, SKS_ZM_NPY=2): a thread owns the two y-adjacent W columns
// (bx, 2g) and (bx, 2g+1), so each column's y neighbour on the other side of the pair comes from
// registers (6 instead of 8 in-plane shared loads per pair and stencil, for U and for the w_j ring)
// and each thread carries two independent FMA chains; 320 threads (10 warps) per CTA.  The kernel is
// latency-bound: measured 36.1 us vs 37.7 us per C3 launch.  Three or six columns per
// thread (a generic version, kept out of the tree) measured 41.2 / 69.4 us: fewer warps, register
// pressure and spills outweigh the saved loads.
static_assert(ZWY % 2 == 0, "the pair kernel needs an even tile height");
constexpr int ZPT = (ZWX * (ZWY / 2) + 31) / 32 * 32;  // 34 x 9 pairs -> 320 threads

// FE (forward-edge, k <= 2 only, default; SKS_ZM_FE=0 turns it off): the second stencil A w_j of phase B is
// replaced by the forward-edge form of the one quadratic form the next step needs,
//     <w, A w> = cc ||w||^2 + (cm + cp) sum_p w_p (w_{p+x} + w_{p+y} + w_{p+z})
// (each edge (p, p+e) contributes w_p cp w_{p+e} from row p and w_{p+e} cm w_p from row p+e; zero Dirichlet values
// outside), and <U, A w_j> is accumulated in phase A as <A^T U, w_j> from the same neighbour sums as A U (reading
// O35); ||A w_j||^2 is not formed (the breakdown reference is derived, reading O39).  Phase B then reads only the
// +x and +y neighbours of w_j from the ring (the +z one is in registers).
#ifndef ZM_NST
#define ZM_NST 3  // TMA stages of the FE pair kernel (3 fit at ZS = 4: 219.5 KB); 2 for the others
#endif
template <int KM, int ZS, bool FE>
__host__ __device__ constexpr int zm_nst() {  // the FE kernel takes ZM_NST stages when they fit
  return (FE && zm_smem_bytes_n<KM, ZS, ZM_NST>() <= 230400) ? ZM_NST : 2;
}
#ifndef ZM_PROD
#define ZM_PROD 1  // 1: an extra (11th) warp issues the TMA stages instead of thread 0 of compute warp 0
#endif
constexpr int ZM_PT = ZM_PROD ? ZPT : 0;          // the issuing thread
constexpr int ZPT_L = ZPT + (ZM_PROD ? 32 : 0);   // threads per CTA of the pair kernel
template <int KM, int ZS, bool FULL, bool USL, bool FE = false>
__global__ void __launch_bounds__(ZPT_L, ZM_CPS)
    step3d_zmp_kernel(StepArgs a, ZmArgs z, const __grid_constant__ CUtensorMap tmU,
                      const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smraw_p[];
  double* sm = reinterpret_cast<double*>(smraw_p + ((128u - (smem_u32(smraw_p) & 127u)) & 127u));
  constexpr int STG = zm_stage<KM, ZS>();
  constexpr int UB = zm_ublk<KM, ZS>(), VB = zm_vblk<KM, ZS>();
  constexpr int R = 3 * ZS;
  constexpr int NST = zm_nst<KM, ZS, FE>();
  double* ring = sm + NST * STG;
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ __align__(8) uint64_t bar[NST];
  const int tid = threadIdx.x;
  if (tid == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    for (int t = 0; t < NST; ++t) mbar_init(&bar[t], 1);
    fence_mbar_init();
  }
  pdl_wait_and_release();
  const int nv = FULL ? KM - 1 : z.nv;  // = cf.nv (host-known), so the first stages can go out now
  const uint32_t sbytes = (uint32_t)(ZUP * (ZS + 2) * 8 + nv * ZVP * ZS * 8);
  const int m = (int)a.m, nz = (int)a.nz, z0g = (int)a.z0, G = a.G;
  const int64_t u_lo = z.use_ub ? (int64_t)z.ub[blockIdx.x] : (z.units * blockIdx.x) / gridDim.x;
  const int64_t u_hi = z.use_ub ? (int64_t)z.ub[blockIdx.x + 1] : (z.units * (blockIdx.x + 1)) / gridDim.x;
  // the first piece's first two stages are issued before the partials reduction of the prologue:
  // their inputs (w_{j-1} and the window) were complete at the PDL wait
  int pre = 0;
  if (ZM_EARLY && tid == ZM_PT && u_lo < u_hi) {
    const int col = (int)(u_lo / nz), za = (int)(u_lo % nz);
    const int64_t zr = za + (u_hi - u_lo);
    const int zb = (int)(zr < nz ? zr : nz);
    const int x0 = (col % z.tiles_x) * ZX, y0 = (col / z.tiles_x) * ZY, wa = za - 1;
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;
    for (int t = 0; t < NST && t < nsteps; ++t) {
      double* dst = sm + t * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[t], sbytes);
      tma_load_4d(dst, &tmU, &bar[t], x0 - 2, y0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB + l * VB, &tmV, &bar[t], x0 - 2, y0 - 1, p0 + G, z.vcol[l]);
      pre = t + 1;
    }
  }
  if (!step_prologue(a, &cf, red)) {
    for (int t = 0; t < pre; ++t) mbar_wait(&bar[t], 0u);  // no bulk copy may outlive the CTA
    return;
  }
  const int64_t pl = a.plane;
  const double cc = a.cc, cm = a.cm, cp = a.cp, alpha = cf.alpha, beta_u = cf.beta_u;
  double cl[KM - 1];
#pragma unroll
  for (int l = 0; l < KM - 1; ++l) cl[l] = (l < nv) ? cf.c[l] : 0.0;
  constexpr bool uslot = USL;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;

  constexpr int NPAIR = ZWX * (ZWY / 2);
  const bool wt = tid < NPAIR;
  const int tp = wt ? tid : NPAIR - 1;
  const int bx = tp % ZWX, by0 = 2 * (tp / ZWX), by1 = by0 + 1;
  const int cu0 = (by0 + 1) * ZUX + (bx + 1), cu1 = cu0 + ZUX;
  const int cv0 = by0 * ZVX + (bx + 1), cv1 = cv0 + ZVX;
  const int cw0 = by0 * ZWX + bx, cw1 = cw0 + ZWX;
  const bool xin_box = bx >= 1 && bx <= ZX;
  const bool in0 = wt && xin_box && by0 >= 1 && by0 <= ZY, in1 = wt && xin_box && by1 >= 1 && by1 <= ZY;

  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;
  uint32_t phase = 0, sidx = 0;
  int carried = pre;  // stages of the coming piece already in flight (thread 0's count)
  for (int64_t u = u_lo; u < u_hi;) {
    const int col = (int)(u / nz);
    const int za = (int)(u % nz);
    const int64_t zr = za + (u_hi - u);
    const int zb = (int)(zr < nz ? zr : nz);
    u += zb - za;
    const int tx = col % z.tiles_x, ty = col / z.tiles_x;
    const int x0 = tx * ZX, y0 = ty * ZY;
    const int wa = za - 1;
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;
    const uint32_t s0 = sidx;
    auto issue = [&](int t) {
      const uint32_t slot = (s0 + (uint32_t)t) % NST;
      double* dst = sm + slot * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[slot], sbytes);
      tma_load_4d(dst, &tmU, &bar[slot], x0 - 2, y0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB + l * VB, &tmV, &bar[slot], x0 - 2, y0 - 1, p0 + G, z.vcol[l]);
    };
    // the next piece (if any): its first two stages go out in the slots freed by this piece's last
    // two steps, so its pipeline fill overlaps this piece's tail
    const bool has_next = u < u_hi;
    const int ncol = has_next ? (int)(u / nz) : 0, nza = has_next ? (int)(u % nz) : 0;
    const int64_t nzr = nza + (u_hi - u);
    const int nzb = (int)(nzr < nz ? nzr : nz);
    const int nx0 = (ncol % z.tiles_x) * ZX, ny0 = (ncol / z.tiles_x) * ZY, nwa = nza - 1;
    const int nnsteps = has_next ? (nzb - nwa + 1 + ZS - 1) / ZS : 0;
    auto issue_next = [&](int tn) {
      const uint32_t slot = (s0 + (uint32_t)nsteps + (uint32_t)tn) % NST;
      double* dst = sm + slot * STG;
      const int p0 = nwa + tn * ZS;
      mbar_arrive_expect_tx(&bar[slot], sbytes);
      tma_load_4d(dst, &tmU, &bar[slot], nx0 - 2, ny0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB + l * VB, &tmV, &bar[slot], nx0 - 2, ny0 - 1, p0 + G, z.vcol[l]);
    };
    if (tid == ZM_PT)
      for (int t = carried; t < NST && t < nsteps; ++t) issue(t);
    carried = 0;
    double wp1a = 0.0, wp2a = 0.0, wp1b = 0.0, wp2b = 0.0;
    double vla[KM - 1], vlb[KM - 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) vla[l] = vlb[l] = 0.0;
    const int gx = x0 - 1 + bx, gy0 = y0 - 1 + by0, gy1 = gy0 + 1;
    const bool xok = wt && (unsigned)gx < (unsigned)m;
    const bool xy0 = xok && (unsigned)gy0 < (unsigned)m, xy1 = xok && (unsigned)gy1 < (unsigned)m;
    const bool aw0 = in0 && gx < m && gy0 < m, aw1 = in1 && gx < m && gy1 < m;
    double* wc0 = Wout + (int64_t)(wa - 1) * pl + (int64_t)gy0 * m + gx;
    double* wc1 = wc0 + m;
    const double am0 = xy0 ? alpha : 0.0, bm0 = xy0 ? beta_u : 0.0;
    const double am1 = xy1 ? alpha : 0.0, bm1 = xy1 ? beta_u : 0.0;
    double clm0[KM - 1], clm1[KM - 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) {
      clm0[l] = xy0 ? cl[l] : 0.0;
      clm1[l] = xy1 ? cl[l] : 0.0;
    }
    constexpr int T0 = ZS == 1 ? 2 : 1;
    auto step = [&](int t, auto phc) {
      constexpr int PH = decltype(phc)::value;
      constexpr int SBW = ((PH + 1) % 3) * ZS;
      constexpr int SBP = SBW == 0 ? R - 1 : SBW - 1;
      const uint32_t slot = (s0 + (uint32_t)t) % NST;
      mbar_wait(&bar[slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
      const double* sU = sm + slot * STG;
      const double* sV = sU + UB;
      const int p0 = wa + t * ZS;
      const bool fast = t >= T0 && p0 + ZS - 1 <= zb && z0g + p0 + ZS - 1 < m;
      double wa_[ZS], wb_[ZS], ca[ZS + 2], cb[ZS + 2], va[KM - 1][ZS], vb[KM - 1][ZS];
      double* rw0 = ring + SBW * ZW + cw0;
      double* rw1 = ring + SBW * ZW + cw1;
      const double* rp0 = ring + SBP * ZW + cw0;
      const double* rp1 = ring + SBP * ZW + cw1;
      if (ZM_PROD && tid >= ZPT) {  // producer warp: no compute
      } else {
#pragma unroll
      for (int k = 0; k < ZS + 2; ++k) {
        ca[k] = sU[k * ZUP + cu0];
        cb[k] = sU[k * ZUP + cu1];
      }
#pragma unroll
      for (int i = 0; i < ZS; ++i) {
        const int p = p0 + i;
#pragma unroll
        for (int l = 0; l < KM - 1; ++l) {
          va[l][i] = (FULL || l < nv) ? sV[l * VB + i * ZVP + cv0] : 0.0;
          vb[l][i] = (FULL || l < nv) ? sV[l * VB + i * ZVP + cv1] : 0.0;
        }
        const double* q0 = sU + (i + 1) * ZUP + cu0;
        const double* q1 = q0 + ZUX;
        // column a (y = by0): y+1 neighbour is column b's centre; column b: y-1 is column a's centre
        const double sma = q0[-1] + q0[-ZUX] + ca[i], spa = q0[1] + cb[i + 1] + ca[i + 2];
        const double smb = q1[-1] + ca[i + 1] + cb[i], spb = q1[1] + q1[ZUX] + cb[i + 2];
        const double Aua = cc * ca[i + 1] + cm * sma + cp * spa;
        const double Aub = cc * cb[i + 1] + cm * smb + cp * spb;
        double w0v, w1v;
        if (fast) {
          w0v = am0 * Aua + bm0 * ca[i + 1];
          w1v = am1 * Aub + bm1 * cb[i + 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (FULL || l < nv) {
              w0v += clm0[l] * va[l][i];
              w1v += clm1[l] * vb[l][i];
            }
        } else {
          w0v = alpha * Aua + beta_u * ca[i + 1];
          w1v = alpha * Aub + beta_u * cb[i + 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (FULL || l < nv) {
              w0v += cl[l] * va[l][i];
              w1v += cl[l] * vb[l][i];
            }
          const bool zok = (unsigned)(z0g + p) < (unsigned)m && p <= zb;
          w0v = (xy0 && zok) ? w0v : 0.0;
          w1v = (xy1 && zok) ? w1v : 0.0;
        }
        wa_[i] = w0v;
        wb_[i] = w1v;
        if (wt) {
          rw0[i * ZW] = w0v;
          rw1[i * ZW] = w1v;
        }
        if constexpr (FE && USL) {  // <U, A w_j> = <A^T U, w_j> on the owned points (plane p in [za, zb))
          const bool zin = p >= za && p < zb;
          const double ta = (aw0 && zin) ? cc * ca[i + 1] + cp * sma + cm * spa : 0.0;
          const double tb = (aw1 && zin) ? cc * cb[i + 1] + cp * smb + cm * spb : 0.0;
          acc[KM + 2] += ta * w0v;
          acc[KM + 2] += tb * w1v;
        }
      }
      }
      __syncthreads();
      if (tid == ZM_PT) {
        if (t + NST < nsteps) {
          issue(t + NST);
        } else if (ZM_NEXT && has_next && nsteps >= NST) {
          const int tn = t + NST - nsteps;  // 0 after step nsteps-NST, ..., NST-1 after the last step
          if (tn < nnsteps) {
            issue_next(tn);
            carried = tn + 1;
          }
        }
      }
      if (aw0 || aw1) {
        double* wo0 = wc0;
        double* wo1 = wc1;
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
          const int qp = p0 - 1 + i;
          if (fast || (qp >= za && qp < zb)) {
            const double wqa = (i == 0) ? wp1a : wa_[i - 1];
            const double wqb = (i == 0) ? wp1b : wb_[i - 1];
            const double wma = (i == 0) ? wp2a : (i == 1 ? wp1a : wa_[i - 2]);
            const double wmb = (i == 0) ? wp2b : (i == 1 ? wp1b : wb_[i - 2]);
            const double* r0 = (i == 0) ? rp0 : rw0 + (i - 1) * ZW;
            const double* r1 = (i == 0) ? rp1 : rw1 + (i - 1) * ZW;
            if constexpr (FE) {
              // forward edges: +x from the ring, +y of a is b's centre, +y of b from the ring, +z in registers
              const double yb = aw1 ? r1[ZWX] : 0.0;
              if (aw0) {
                *wo0 = wqa;
                acc[0] += wqa * wqa;
                acc[2] += wqa * (r0[1] + wqb + wa_[i]);
              }
              if (aw1) {
                *wo1 = wqb;
                acc[0] += wqb * wqb;
                acc[2] += wqb * (r1[1] + yb + wb_[i]);
              }
              (void)wma;
              (void)wmb;
              wo0 += pl;
              wo1 += pl;
              continue;
            }
            // the pair's outer y neighbours are read only for an output column (the row past the
            // last W row lies outside the ring)
            const double ya = aw0 ? r0[-ZWX] : 0.0, yb = aw1 ? r1[ZWX] : 0.0;
            const double Awa = cc * wqa + cm * (r0[-1] + ya + wma) + cp * (r0[1] + wqb + wa_[i]);
            const double Awb = cc * wqb + cm * (r1[-1] + wqa + wmb) + cp * (r1[1] + yb + wb_[i]);
            if (aw0) {
              *wo0 = wqa;
              acc[0] += wqa * wqa;
              acc[1] += wqa * Awa;
              acc[2] += Awa * Awa;
              if (uslot) acc[KM + 2] += ca[i] * Awa;
#pragma unroll
              for (int l = 0; l < KM - 1; ++l)
                if (FULL || l < nv) acc[3 + l] += ((i == 0) ? vla[l] : va[l][i - 1]) * Awa;
            }
            if (aw1) {
              *wo1 = wqb;
              acc[0] += wqb * wqb;
              acc[1] += wqb * Awb;
              acc[2] += Awb * Awb;
              if (uslot) acc[KM + 2] += cb[i] * Awb;
#pragma unroll
              for (int l = 0; l < KM - 1; ++l)
                if (FULL || l < nv) acc[3 + l] += ((i == 0) ? vlb[l] : vb[l][i - 1]) * Awb;
            }
          }
          wo0 += pl;
          wo1 += pl;
        }
      }
      wp2a = ZS >= 2 ? wa_[ZS >= 2 ? ZS - 2 : 0] : wp1a;
      wp2b = ZS >= 2 ? wb_[ZS >= 2 ? ZS - 2 : 0] : wp1b;
      wp1a = wa_[ZS - 1];
      wp1b = wb_[ZS - 1];
#pragma unroll
      for (int l = 0; l < KM - 1; ++l) {
        vla[l] = va[l][ZS - 1];
        vlb[l] = vb[l][ZS - 1];
      }
      wc0 += (int64_t)ZS * pl;
      wc1 += (int64_t)ZS * pl;
    };
    for (int t = 0; t < nsteps; t += 3) {
      step(t, std::integral_constant<int, 0>{});
      if (t + 1 < nsteps) step(t + 1, std::integral_constant<int, 1>{});
      if (t + 2 < nsteps) step(t + 2, std::integral_constant<int, 2>{});
    }
    sidx = s0 + (uint32_t)nsteps;
    __syncthreads();
  }
  if constexpr (FE) {  // slot 1: <w, A w> from ||w||^2 and the forward-edge sum; slot 2 (||A w||^2) is not formed
    acc[1] = cc * acc[0] + (cm + cp) * acc[2];
    acc[2] = 0.0;
  }
  step_epilogue<KM>(a, &cf, acc, red);
}


// ---- plane-split forward-edge kernel (opt-in SKS_ZM_NG=2; measured slower: 38.8 vs 31.6 us at C3, 96 registers with spills).
// The FE pair kernel runs 10 warps per SM (150 registers) and is latency-bound: each warp walks the ZS planes of a
// step as one long dependent stream.  Here NG thread groups share a step: group g owns planes [g H, (g+1) H) of the
// step (H = ZS / NG) for the same 34 x 9 pairs, so the SM holds NG x 10 warps with the same stages and ring.  Phase A
// of group g reads its U planes p-1 .. p+H from the stage; phase B of group g needs w_j at its planes q = p-1 ..
// p+H-2 and the +z neighbour q+1 (own registers), except that the first plane q = p-1 of a group was formed by the
// group (or step) before it and is read from the ring.  Arithmetic per point is that of the FE pair kernel.
template <int ZS, int NG, bool FULL, bool USL>
__global__ void __launch_bounds__(ZPT * NG, 1)
    step3d_zfe_kernel(StepArgs a, ZmArgs z, const __grid_constant__ CUtensorMap tmU,
                      const __grid_constant__ CUtensorMap tmV) {
  constexpr int KM = 2;
  constexpr int H = ZS / NG;
  static_assert(ZS % NG == 0, "planes per step must split evenly over the groups");
  extern __shared__ __align__(128) unsigned char smraw_f[];
  double* sm = reinterpret_cast<double*>(smraw_f + ((128u - (smem_u32(smraw_f) & 127u)) & 127u));
  constexpr int STG = zm_stage<KM, ZS>();
  constexpr int UB = zm_ublk<KM, ZS>();
  constexpr int R = 3 * ZS;
  double* ring = sm + 2 * STG;
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ __align__(8) uint64_t bar[2];
  const int tid = threadIdx.x;
  if (tid == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  pdl_wait_and_release();
  const int nv = FULL ? KM - 1 : z.nv;
  const uint32_t sbytes = (uint32_t)(ZUP * (ZS + 2) * 8 + nv * ZVP * ZS * 8);
  const int m = (int)a.m, nz = (int)a.nz, z0g = (int)a.z0, G = a.G;
  const int64_t u_lo = z.use_ub ? (int64_t)z.ub[blockIdx.x] : (z.units * blockIdx.x) / gridDim.x;
  const int64_t u_hi = z.use_ub ? (int64_t)z.ub[blockIdx.x + 1] : (z.units * (blockIdx.x + 1)) / gridDim.x;
  int pre = 0;
  if (ZM_EARLY && tid == 0 && u_lo < u_hi) {
    const int col = (int)(u_lo / nz), za = (int)(u_lo % nz);
    const int64_t zr = za + (u_hi - u_lo);
    const int zb = (int)(zr < nz ? zr : nz);
    const int x0 = (col % z.tiles_x) * ZX, y0 = (col / z.tiles_x) * ZY, wa = za - 1;
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;
    for (int t = 0; t < 2 && t < nsteps; ++t) {
      double* dst = sm + t * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[t], sbytes);
      tma_load_4d(dst, &tmU, &bar[t], x0 - 2, y0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB, &tmV, &bar[t], x0 - 2, y0 - 1, p0 + G, z.vcol[l]);
      pre = t + 1;
    }
  }
  if (!step_prologue(a, &cf, red)) {
    for (int t = 0; t < pre; ++t) mbar_wait(&bar[t], 0u);
    return;
  }
  const int64_t pl = a.plane;
  const double cc = a.cc, cm = a.cm, cp = a.cp, alpha = cf.alpha, beta_u = cf.beta_u;
  const double cl = (nv > 0) ? cf.c[0] : 0.0;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;

  constexpr int NPAIR = ZWX * (ZWY / 2);
  const int grp = tid / ZPT, tin = tid - grp * ZPT;
  const int i0 = grp * H;  // first plane (within a step) of this group
  const bool wt = tin < NPAIR;
  const int tp = wt ? tin : NPAIR - 1;
  const int bx = tp % ZWX, by0 = 2 * (tp / ZWX), by1 = by0 + 1;
  const int cu0 = (by0 + 1) * ZUX + (bx + 1), cu1 = cu0 + ZUX;
  const int cv0 = by0 * ZVX + (bx + 1), cv1 = cv0 + ZVX;
  const int cw0 = by0 * ZWX + bx, cw1 = cw0 + ZWX;
  const bool xin_box = bx >= 1 && bx <= ZX;
  const bool in0 = wt && xin_box && by0 >= 1 && by0 <= ZY, in1 = wt && xin_box && by1 >= 1 && by1 <= ZY;

  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;
  uint32_t phase = 0, sidx = 0;
  int carried = pre;
  for (int64_t u = u_lo; u < u_hi;) {
    const int col = (int)(u / nz);
    const int za = (int)(u % nz);
    const int64_t zr = za + (u_hi - u);
    const int zb = (int)(zr < nz ? zr : nz);
    u += zb - za;
    const int tx = col % z.tiles_x, ty = col / z.tiles_x;
    const int x0 = tx * ZX, y0 = ty * ZY;
    const int wa = za - 1;
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;
    const uint32_t s0 = sidx;
    auto issue = [&](int t) {
      const uint32_t slot = (s0 + (uint32_t)t) & 1u;
      double* dst = sm + slot * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[slot], sbytes);
      tma_load_4d(dst, &tmU, &bar[slot], x0 - 2, y0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB, &tmV, &bar[slot], x0 - 2, y0 - 1, p0 + G, z.vcol[l]);
    };
    const bool has_next = u < u_hi;
    const int ncol = has_next ? (int)(u / nz) : 0, nza = has_next ? (int)(u % nz) : 0;
    const int64_t nzr = nza + (u_hi - u);
    const int nzb = (int)(nzr < nz ? nzr : nz);
    const int nx0 = (ncol % z.tiles_x) * ZX, ny0 = (ncol / z.tiles_x) * ZY, nwa = nza - 1;
    const int nnsteps = has_next ? (nzb - nwa + 1 + ZS - 1) / ZS : 0;
    auto issue_next = [&](int tn) {
      const uint32_t slot = (s0 + (uint32_t)nsteps + (uint32_t)tn) & 1u;
      double* dst = sm + slot * STG;
      const int p0 = nwa + tn * ZS;
      mbar_arrive_expect_tx(&bar[slot], sbytes);
      tma_load_4d(dst, &tmU, &bar[slot], nx0 - 2, ny0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_4d(dst + UB, &tmV, &bar[slot], nx0 - 2, ny0 - 1, p0 + G, z.vcol[l]);
    };
    if (tid == 0)
      for (int t = carried; t < 2 && t < nsteps; ++t) issue(t);
    carried = 0;
    const int gx = x0 - 1 + bx, gy0 = y0 - 1 + by0, gy1 = gy0 + 1;
    const bool xok = wt && (unsigned)gx < (unsigned)m;
    const bool xy0 = xok && (unsigned)gy0 < (unsigned)m, xy1 = xok && (unsigned)gy1 < (unsigned)m;
    const bool aw0 = in0 && gx < m && gy0 < m, aw1 = in1 && gx < m && gy1 < m;
    // global output of this group's first phase-B plane q = p0 - 1 + i0 (step 0)
    double* wc0 = Wout + (int64_t)(wa - 1 + i0) * pl + (int64_t)gy0 * m + gx;
    double* wc1 = wc0 + m;
    const double am0 = xy0 ? alpha : 0.0, bm0 = xy0 ? beta_u : 0.0, clm0 = xy0 ? cl : 0.0;
    const double am1 = xy1 ? alpha : 0.0, bm1 = xy1 ? beta_u : 0.0, clm1 = xy1 ? cl : 0.0;
    constexpr int T0 = ZS == 1 ? 2 : 1;
    auto step = [&](int t, auto phc) {
      constexpr int PH = decltype(phc)::value;
      constexpr int SBW = ((PH + 1) % 3) * ZS;
      constexpr int SBP = SBW == 0 ? R - 1 : SBW - 1;
      const uint32_t slot = (s0 + (uint32_t)t) & 1u;
      mbar_wait(&bar[slot], (phase >> slot) & 1u);
      phase ^= 1u << slot;
      const double* sU = sm + slot * STG;
      const double* sV = sU + UB;
      const int p0 = wa + t * ZS;
      const int pg = p0 + i0;  // this group's first plane
      const bool fast = t >= T0 && p0 + ZS - 1 <= zb && z0g + p0 + ZS - 1 < m;
      double wa_[H], wb_[H], ca[H + 2], cb[H + 2], va[H], vb[H];
      double* rw0 = ring + SBW * ZW + i0 * ZW + cw0;
      double* rw1 = ring + SBW * ZW + i0 * ZW + cw1;
#pragma unroll
      for (int k = 0; k < H + 2; ++k) {
        ca[k] = sU[(i0 + k) * ZUP + cu0];
        cb[k] = sU[(i0 + k) * ZUP + cu1];
      }
#pragma unroll
      for (int ii = 0; ii < H; ++ii) {
        const int p = pg + ii;
        va[ii] = (FULL || nv > 0) ? sV[(i0 + ii) * ZVP + cv0] : 0.0;
        vb[ii] = (FULL || nv > 0) ? sV[(i0 + ii) * ZVP + cv1] : 0.0;
        const double* q0 = sU + (i0 + ii + 1) * ZUP + cu0;
        const double* q1 = q0 + ZUX;
        const double sma = q0[-1] + q0[-ZUX] + ca[ii], spa = q0[1] + cb[ii + 1] + ca[ii + 2];
        const double smb = q1[-1] + ca[ii + 1] + cb[ii], spb = q1[1] + q1[ZUX] + cb[ii + 2];
        const double Aua = cc * ca[ii + 1] + cm * sma + cp * spa;
        const double Aub = cc * cb[ii + 1] + cm * smb + cp * spb;
        double w0v, w1v;
        if (fast) {
          w0v = am0 * Aua + bm0 * ca[ii + 1];
          w1v = am1 * Aub + bm1 * cb[ii + 1];
          if (FULL || nv > 0) {
            w0v += clm0 * va[ii];
            w1v += clm1 * vb[ii];
          }
        } else {
          w0v = alpha * Aua + beta_u * ca[ii + 1];
          w1v = alpha * Aub + beta_u * cb[ii + 1];
          if (FULL || nv > 0) {
            w0v += cl * va[ii];
            w1v += cl * vb[ii];
          }
          const bool zok = (unsigned)(z0g + p) < (unsigned)m && p <= zb;
          w0v = (xy0 && zok) ? w0v : 0.0;
          w1v = (xy1 && zok) ? w1v : 0.0;
        }
        wa_[ii] = w0v;
        wb_[ii] = w1v;
        if (wt) {
          rw0[ii * ZW] = w0v;
          rw1[ii * ZW] = w1v;
        }
        if constexpr (USL) {  // <U, A w_j> = <A^T U, w_j> on the owned points (plane p in [za, zb))
          const bool zin = p >= za && p < zb;
          const double ta = (aw0 && zin) ? cc * ca[ii + 1] + cp * sma + cm * spa : 0.0;
          const double tb = (aw1 && zin) ? cc * cb[ii + 1] + cp * smb + cm * spb : 0.0;
          acc[KM + 2] += ta * w0v;
          acc[KM + 2] += tb * w1v;
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (t + 2 < nsteps) {
          issue(t + 2);
        } else if (ZM_NEXT && has_next && nsteps >= 2) {
          const int tn = t + 2 - nsteps;
          if (tn < nnsteps) {
            issue_next(tn);
            carried = tn + 1;
          }
        }
      }
      if (aw0 || aw1) {
        // the group's first phase-B plane q = pg - 1: formed by the previous group (this step's ring) or, for group 0,
        // by the last group of the previous step (the previous segment's last plane)
        const double* rf0 = (i0 == 0) ? ring + SBP * ZW + cw0 : rw0 - ZW;
        const double* rf1 = (i0 == 0) ? ring + SBP * ZW + cw1 : rw1 - ZW;
        double* wo0 = wc0;
        double* wo1 = wc1;
#pragma unroll
        for (int ii = 0; ii < H; ++ii) {
          const int qp = pg - 1 + ii;
          if (fast || (qp >= za && qp < zb)) {
            const double* r0 = (ii == 0) ? rf0 : rw0 + (ii - 1) * ZW;
            const double* r1 = (ii == 0) ? rf1 : rw1 + (ii - 1) * ZW;
            const double wqa = (ii == 0) ? r0[0] : wa_[ii - 1];
            const double wqb = (ii == 0) ? r1[0] : wb_[ii - 1];
            const double yb = aw1 ? r1[ZWX] : 0.0;
            if (aw0) {
              *wo0 = wqa;
              acc[0] += wqa * wqa;
              acc[2] += wqa * (r0[1] + wqb + wa_[ii]);
            }
            if (aw1) {
              *wo1 = wqb;
              acc[0] += wqb * wqb;
              acc[2] += wqb * (r1[1] + yb + wb_[ii]);
            }
          }
          wo0 += pl;
          wo1 += pl;
        }
      }
      wc0 += (int64_t)ZS * pl;
      wc1 += (int64_t)ZS * pl;
    };
    for (int t = 0; t < nsteps; t += 3) {
      step(t, std::integral_constant<int, 0>{});
      if (t + 1 < nsteps) step(t + 1, std::integral_constant<int, 1>{});
      if (t + 2 < nsteps) step(t + 2, std::integral_constant<int, 2>{});
    }
    sidx = s0 + (uint32_t)nsteps;
    __syncthreads();
  }
  acc[1] = cc * acc[0] + (cm + cp) * acc[2];  // <w, A w> from ||w||^2 and the forward-edge sum (reading O39)
  acc[2] = 0.0;
  step_epilogue<KM>(a, &cf, acc, red);
}

// ---- warp-specialised variant (SKS_ZM_WS=1; measured 37.5 us vs 35.1 us for the pair kernel at C3, so the
// pair kernel stays the default -- DESIGN.md section 11).
// The pair kernel runs its two phases -- (A) w_j on the W box from the staged U/V planes, (B) A w_j and the
// next step's dot products on the interior -- on the same 10 warps with a CTA barrier between them, so each
// phase's FP64 and shared-memory latencies are exposed (ncu r01j: 'wait' and 'short_scoreboard' stalls, issue
// active 29%).  Here the phases run on two warp groups, one step apart, handing the w_j ring over through
// mbarriers (no CTA-wide barrier inside the march):
//   group A (10 warps, pairs of the 34 x 18 W box): waits for the stage (TMA) and for the ring segment to be
//     free, forms w_j for ZS planes, writes the ring segment and the interior w_j to global memory;
//     it also accumulates <U, A w_j> as <A^T U, w_j> (A^T u from the same neighbour sums as A u, reading O35)
//     and its thread 0 refills a stage once all group-A warps have released it;
//   group B (8 warps, pairs of the 32 x 16 interior): waits for the ring segment, forms A w_j from the ring
//     (z neighbours carried in registers) and accumulates ||w||^2, <w,Aw>, ||Aw||^2 and the window dots
//     <V_l,Aw> (read from the stage; none for k = 2, where group B never touches the stages).
// Stages: NST = 3 when they fit (k = 2), else 2.  Ring: 3 segments of ZS planes; segment g mod 3 is written
// by A at global step g and read by B at steps g and g+1, so A may run up to two steps ahead of B.
#ifndef ZWS_SLEEP_B
#define ZWS_SLEEP_B 0  // suspend-time hint (ns) of group B's ring wait (0: plain try_wait)
#endif
#ifndef ZWS_SLEEP_A
#define ZWS_SLEEP_A 0
#endif
constexpr int WA_T = 320;                 // group A threads (34 x 9 = 306 pairs used)
constexpr int WB_T = 256;                 // group B threads (32 x 8 pairs)
constexpr int WS_T = WA_T + WB_T;         // 18 warps
template <int KM, int ZS, int NST>
__host__ __device__ constexpr size_t zws_smem_bytes() {
  return 128 + sizeof(double) * ((size_t)NST * zm_stage<KM, ZS>() + (size_t)(3 * ZS) * ZW);
}

struct ZPiece {
  int za, zb, x0, y0, wa, nsteps;
};
template <int ZS>
__device__ __forceinline__ ZPiece zws_piece(const ZmArgs& z, int nz, int64_t u, int64_t u_hi) {
  ZPiece p;
  const int col = (int)(u / nz);
  p.za = (int)(u % nz);
  const int64_t zr = p.za + (u_hi - u);
  p.zb = (int)(zr < nz ? zr : nz);
  p.x0 = (col % z.tiles_x) * ZX;
  p.y0 = (col / z.tiles_x) * ZY;
  p.wa = p.za - 1;
  p.nsteps = (p.zb - p.wa + 1 + ZS - 1) / ZS;
  return p;
}
// walks the (piece, step) sequence of one CTA
template <int ZS>
struct ZCursor {
  int64_t u, u_hi;
  ZPiece pc;
  int t;
  bool valid;
  __device__ __forceinline__ void init(const ZmArgs& z, int nz, int64_t lo, int64_t hi) {
    u = lo;
    u_hi = hi;
    t = 0;
    valid = u < u_hi;
    if (valid) pc = zws_piece<ZS>(z, nz, u, u_hi);
  }
  __device__ __forceinline__ void next_piece(const ZmArgs& z, int nz) {
    u += pc.zb - pc.za;
    t = 0;
    valid = u < u_hi;
    if (valid) pc = zws_piece<ZS>(z, nz, u, u_hi);
  }
  __device__ __forceinline__ void next(const ZmArgs& z, int nz) {
    if (++t >= pc.nsteps) next_piece(z, nz);
  }
};

template <int KM, int ZS, int NST, bool FULL, bool USL>
__global__ void __launch_bounds__(WS_T, 1)
    step3d_zws_kernel(StepArgs a, ZmArgs z, const __grid_constant__ CUtensorMap tmU,
                      const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smraw_w[];
  double* sm = reinterpret_cast<double*>(smraw_w + ((128u - (smem_u32(smraw_w) & 127u)) & 127u));
  constexpr int STG = zm_stage<KM, ZS>();
  constexpr int UB = zm_ublk<KM, ZS>(), VB = zm_vblk<KM, ZS>();
  constexpr int SEG = ZS * ZW;  // doubles per ring segment
  double* ring = sm + NST * STG;
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ __align__(8) uint64_t full[NST], sempty[NST], rfull[3], rempty[3];
  const int tid = threadIdx.x, lane = tid & 31;
  if (tid == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    for (int i = 0; i < NST; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&sempty[i], (WA_T + (z.vdot ? WB_T : 0)) / 32);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&rfull[i], WA_T / 32);
      mbar_init(&rempty[i], WB_T / 32);
    }
    fence_mbar_init();
  }
  pdl_wait_and_release();
  const int nv = FULL ? KM - 1 : z.nv;
  const uint32_t sbytes = (uint32_t)(ZUP * (ZS + 2) * 8 + nv * ZVP * ZS * 8);
  const int m = (int)a.m, nz = (int)a.nz, z0g = (int)a.z0, G = a.G;
  const int64_t u_lo = z.use_ub ? (int64_t)z.ub[blockIdx.x] : (z.units * blockIdx.x) / gridDim.x;
  const int64_t u_hi = z.use_ub ? (int64_t)z.ub[blockIdx.x + 1] : (z.units * (blockIdx.x + 1)) / gridDim.x;
  auto issue = [&](const ZCursor<ZS>& c, int slot) {
    double* dst = sm + slot * STG;
    const int p0 = c.pc.wa + c.t * ZS;
    mbar_arrive_expect_tx(&full[slot], sbytes);
    tma_load_4d(dst, &tmU, &full[slot], c.pc.x0 - 2, c.pc.y0 - 2, p0 - 1 + G, z.ucol);
    for (int l = 0; l < nv; ++l)
      tma_load_4d(dst + UB + l * VB, &tmV, &full[slot], c.pc.x0 - 2, c.pc.y0 - 1, p0 + G, z.vcol[l]);
  };
  // the first NST stages go out before the prologue's partials reduction (inputs complete at the PDL wait)
  int pre = 0;
  if (tid == 0) {
    ZCursor<ZS> c;
    c.init(z, nz, u_lo, u_hi);
    for (; pre < NST && c.valid; ++pre) {
      issue(c, pre);
      c.next(z, nz);
    }
  }
  if (!step_prologue(a, &cf, red)) {
    if (tid == 0)
      for (int t = 0; t < pre; ++t) mbar_wait(&full[t], 0u);  // no bulk copy may outlive the CTA
    return;
  }
  const double cc = a.cc, cm = a.cm, cp = a.cp;
  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;

  if (tid < WA_T) {
    // ======================= group A: w_j on the W box ========================================
    const int64_t pl = a.plane;
    const double alpha = cf.alpha, beta_u = cf.beta_u;
    double cl[KM - 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) cl[l] = (l < nv) ? cf.c[l] : 0.0;
    double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;
    constexpr int NPAIR = ZWX * (ZWY / 2);
    const bool wt = tid < NPAIR;
    const int tp = wt ? tid : NPAIR - 1;
    const int bx = tp % ZWX, by0 = 2 * (tp / ZWX), by1 = by0 + 1;
    const int cu0 = (by0 + 1) * ZUX + (bx + 1), cu1 = cu0 + ZUX;
    const int cv0 = by0 * ZVX + (bx + 1), cv1 = cv0 + ZVX;
    const int cw0 = by0 * ZWX + bx, cw1 = cw0 + ZWX;
    const bool xin_box = bx >= 1 && bx <= ZX;
    const bool in0 = wt && xin_box && by0 >= 1 && by0 <= ZY, in1 = wt && xin_box && by1 >= 1 && by1 <= ZY;
    uint32_t g = 0;
    ZCursor<ZS> cur, ahead;  // ahead: the stage warp 0 issues next (global step g + NST)
    cur.init(z, nz, u_lo, u_hi);
    const bool producer = tid == 0;
    if (producer) {
      ahead.init(z, nz, u_lo, u_hi);
      for (int i = 0; i < NST && ahead.valid; ++i) ahead.next(z, nz);
    }
    while (cur.valid) {
      const ZPiece pc = cur.pc;
      const int gx = pc.x0 - 1 + bx, gy0 = pc.y0 - 1 + by0, gy1 = gy0 + 1;
      const bool xok = wt && (unsigned)gx < (unsigned)m;
      const bool xy0 = xok && (unsigned)gy0 < (unsigned)m, xy1 = xok && (unsigned)gy1 < (unsigned)m;
      const bool st0 = in0 && gx < m && gy0 < m, st1 = in1 && gx < m && gy1 < m;
      double* wc0 = Wout + (int64_t)gy0 * m + gx;
      double* wc1 = wc0 + m;
      const double am0 = xy0 ? alpha : 0.0, bm0 = xy0 ? beta_u : 0.0;
      const double am1 = xy1 ? alpha : 0.0, bm1 = xy1 ? beta_u : 0.0;
      double clm0[KM - 1], clm1[KM - 1];
#pragma unroll
      for (int l = 0; l < KM - 1; ++l) {
        clm0[l] = xy0 ? cl[l] : 0.0;
        clm1[l] = xy1 ? cl[l] : 0.0;
      }
      constexpr int T0 = ZS == 1 ? 2 : 1;
      for (int t = 0; t < pc.nsteps; ++t, ++g) {
        const int slot = (int)(g % NST), seg = (int)(g % 3);
        mbar_wait(&full[slot], (g / NST) & 1u);
        if (g >= 3) mbar_wait_sleep(&rempty[seg], ((g / 3) - 1) & 1u, ZWS_SLEEP_A);
        const double* sU = sm + slot * STG;
        const double* sV = sU + UB;
        const int p0 = pc.wa + t * ZS;
        const bool fast = t >= T0 && p0 + ZS - 1 <= pc.zb && z0g + p0 + ZS - 1 < m;
        double ca[ZS + 2], cb[ZS + 2];
        double* rw0 = ring + seg * SEG + cw0;
        double* rw1 = ring + seg * SEG + cw1;
#pragma unroll
        for (int k = 0; k < ZS + 2; ++k) {
          ca[k] = sU[k * ZUP + cu0];
          cb[k] = sU[k * ZUP + cu1];
        }
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
          const int p = p0 + i;
          double va[KM - 1], vb[KM - 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l) {
            va[l] = (FULL || l < nv) ? sV[l * VB + i * ZVP + cv0] : 0.0;
            vb[l] = (FULL || l < nv) ? sV[l * VB + i * ZVP + cv1] : 0.0;
          }
          const double* q0 = sU + (i + 1) * ZUP + cu0;
          const double* q1 = q0 + ZUX;
          // minus / plus neighbour sums of U; A u = cc u + cm sM + cp sP and (transposed convection)
          // A^T u = cc u + cp sM + cm sP, so <U, A w> = <A^T U, w> is accumulated here, on the points this
          // thread stores, and group B never reads the stage (reading O35)
          const double sMa = q0[-1] + q0[-ZUX] + ca[i], sPa = q0[1] + cb[i + 1] + ca[i + 2];
          const double sMb = q1[-1] + ca[i + 1] + cb[i], sPb = q1[1] + q1[ZUX] + cb[i + 2];
          const double Aua = cc * ca[i + 1] + cm * sMa + cp * sPa;
          const double Aub = cc * cb[i + 1] + cm * sMb + cp * sPb;
          double w0v, w1v;
          if (fast) {
            w0v = am0 * Aua + bm0 * ca[i + 1];
            w1v = am1 * Aub + bm1 * cb[i + 1];
#pragma unroll
            for (int l = 0; l < KM - 1; ++l)
              if (FULL || l < nv) {
                w0v += clm0[l] * va[l];
                w1v += clm1[l] * vb[l];
              }
          } else {
            w0v = alpha * Aua + beta_u * ca[i + 1];
            w1v = alpha * Aub + beta_u * cb[i + 1];
#pragma unroll
            for (int l = 0; l < KM - 1; ++l)
              if (FULL || l < nv) {
                w0v += cl[l] * va[l];
                w1v += cl[l] * vb[l];
              }
            const bool zok = (unsigned)(z0g + p) < (unsigned)m && p <= pc.zb;
            w0v = (xy0 && zok) ? w0v : 0.0;
            w1v = (xy1 && zok) ? w1v : 0.0;
          }
          if (wt) {
            rw0[i * ZW] = w0v;
            rw1[i * ZW] = w1v;
          }
          // the output planes [za, zb) of w_j (a fast step has p >= za; only its last plane can be zb)
          if (fast ? (i < ZS - 1 || p < pc.zb) : (p >= pc.za && p < pc.zb)) {
            if (st0) {
              if (!z.store_b) wc0[(int64_t)p * pl] = w0v;
              if (USL) acc[KM + 2] += (cc * ca[i + 1] + cp * sMa + cm * sPa) * w0v;
            }
            if (st1) {
              if (!z.store_b) wc1[(int64_t)p * pl] = w1v;
              if (USL) acc[KM + 2] += (cc * cb[i + 1] + cp * sMb + cm * sPb) * w1v;
            }
          }
        }
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&rfull[seg]);
          mbar_arrive(&sempty[slot]);
        }
        if (producer && ahead.valid) {  // refill this slot with global step g + NST once it is released
          mbar_wait(&sempty[slot], (g / NST) & 1u);
          issue(ahead, slot);
          ahead.next(z, nz);
        }
      }
      cur.next_piece(z, nz);
    }
  } else {
    // ======================= group B: A w_j and the next step's dot products =====================
    const int tb = tid - WA_T;
    const int bx = 1 + tb % ZX, by0 = 1 + 2 * (tb / ZX);
    const int cv0 = by0 * ZVX + (bx + 1), cv1 = cv0 + ZVX;
    const int cw0 = by0 * ZWX + bx, cw1 = cw0 + ZWX;
    const int vdot = z.vdot;
    uint32_t g = 0;
    ZCursor<ZS> cur;
    cur.init(z, nz, u_lo, u_hi);
    while (cur.valid) {
      const ZPiece pc = cur.pc;
      const int gx = pc.x0 - 1 + bx, gy0 = pc.y0 - 1 + by0, gy1 = gy0 + 1;
      const bool aw0 = gx < m && gy0 < m, aw1 = gx < m && gy1 < m;
      const bool sb = z.store_b != 0;
      double* wo0 = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off + (int64_t)gy0 * m + gx;
      double* wo1 = wo0 + m;
      double wm1a = 0.0, w0a = 0.0, wm1b = 0.0, w0b = 0.0;  // w_j at planes p0-2, p0-1 (carried)
      double vla[KM - 1], vlb[KM - 1];
#pragma unroll
      for (int l = 0; l < KM - 1; ++l) vla[l] = vlb[l] = 0.0;
      constexpr int T0 = ZS == 1 ? 2 : 1;
      for (int t = 0; t < pc.nsteps; ++t, ++g) {
        const int slot = (int)(g % NST), seg = (int)(g % 3), sprev = (int)((g + 2) % 3);
        if (vdot) mbar_wait(&full[slot], (g / NST) & 1u);  // the stage is read only for window dots
        mbar_wait_sleep(&rfull[seg], (g / 3) & 1u, ZWS_SLEEP_B);
        const double* sU = sm + slot * STG;
        const double* sV = sU + UB;
        const int p0 = pc.wa + t * ZS;
        const bool fast = t >= T0 && p0 + ZS - 1 <= pc.zb && z0g + p0 + ZS - 1 < m;
        const double* rs = ring + seg * SEG;
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
          const int qp = p0 - 1 + i;
          const double* rq = (i == 0) ? ring + sprev * SEG + (ZS - 1) * ZW : rs + (i - 1) * ZW;  // plane qp
          const double wp1a = rs[i * ZW + cw0], wp1b = rs[i * ZW + cw1];                       // plane qp + 1
          const double Awa = cc * w0a + cm * (rq[cw0 - 1] + rq[cw0 - ZWX] + wm1a) + cp * (rq[cw0 + 1] + w0b + wp1a);
          const double Awb = cc * w0b + cm * (rq[cw1 - 1] + w0a + wm1b) + cp * (rq[cw1 + 1] + rq[cw1 + ZWX] + wp1b);
          if (fast || (qp >= pc.za && qp < pc.zb)) {
            if (sb) {
              if (aw0) wo0[(int64_t)qp * a.plane] = w0a;
              if (aw1) wo1[(int64_t)qp * a.plane] = w0b;
            }
            if (aw0) {
              acc[0] += w0a * w0a;
              acc[1] += w0a * Awa;
              acc[2] += Awa * Awa;
#pragma unroll
              for (int l = 0; l < KM - 1; ++l)
                if ((FULL || l < nv) && ((vdot >> l) & 1))
                  acc[3 + l] += ((i == 0) ? vla[l] : sV[l * VB + (i - 1) * ZVP + cv0]) * Awa;
            }
            if (aw1) {
              acc[0] += w0b * w0b;
              acc[1] += w0b * Awb;
              acc[2] += Awb * Awb;
#pragma unroll
              for (int l = 0; l < KM - 1; ++l)
                if ((FULL || l < nv) && ((vdot >> l) & 1))
                  acc[3 + l] += ((i == 0) ? vlb[l] : sV[l * VB + (i - 1) * ZVP + cv1]) * Awb;
            }
          }
          wm1a = w0a;
          w0a = wp1a;
          wm1b = w0b;
          w0b = wp1b;
        }
#pragma unroll
        for (int l = 0; l < KM - 1; ++l)
          if ((FULL || l < nv) && ((vdot >> l) & 1)) {
            vla[l] = sV[l * VB + (ZS - 1) * ZVP + cv0];
            vlb[l] = sV[l * VB + (ZS - 1) * ZVP + cv1];
          }
        __syncwarp();
        if (lane == 0) {
          if (vdot) mbar_arrive(&sempty[slot]);
          if (g >= 1) mbar_arrive(&rempty[sprev]);
        }
      }
      cur.next_piece(z, nz);
    }
  }
  __syncthreads();
  step_epilogue<KM>(a, &cf, acc, red);
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_enc_zm = nullptr;

static bool zm_encode_fn() {
  if (g_enc_zm) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_enc_zm = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// 4D map {x: m, y: m, z_storage: nz+2G, column: ncol} over columns of pitch ld; one plane per box
static bool zm_encode(CUtensorMap* out, const double* base, int64_t m, int64_t nz, int G, int64_t ld, int64_t ncol,
                      bool ubox, int bdepth) {
  if (!zm_encode_fn()) return false;
  cuuint64_t dims[4] = {(cuuint64_t)m, (cuuint64_t)m, (cuuint64_t)(nz + 2 * G), (cuuint64_t)ncol};
  cuuint64_t strides[3] = {(cuuint64_t)(m * 8), (cuuint64_t)(m * m * 8), (cuuint64_t)(ld * 8)};
  cuuint32_t box[4] = {(cuuint32_t)(ubox ? ZUX : ZVX), (cuuint32_t)(ubox ? ZUY : ZVY), (cuuint32_t)bdepth, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = g_enc_zm(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct ZmMaps {
  CUtensorMap WU, WV, XU, FV, VU;
  MapKey key[5];
  int64_t part_key = -1;  // step-balanced partition cache
  bool part_ok = false;
  int32_t ub[ZM_MAXG + 1];
};

template <int KM>
constexpr int zm_zs() {
  constexpr size_t cap = (ZM_CPS > 1 ? 226 * 1024 / ZM_CPS - 1024 : 200 * 1024);
#ifdef ZM_ZS  // experiment: planes per step (falls back when the stages do not fit)
  if (zm_smem_bytes<KM, ZM_ZS>() <= 226 * 1024 / ZM_CPS - 1024) return ZM_ZS;
#endif
  return zm_smem_bytes<KM, 4>() <= cap ? 4 : (zm_smem_bytes<KM, 2>() <= cap ? 2 : 1);
}

static int zm_npy() {  // W columns per thread: 1 = step3d_zm_kernel, 2 = step3d_zmp_kernel (SKS_ZM_NPY)
  static int npy = -1;
  if (npy < 0) {
    const char* e = getenv("SKS_ZM_NPY");
    npy = e ? atoi(e) : ZM_NPY_DEFAULT;
    if (npy != 1 && npy != 2) npy = ZM_NPY_DEFAULT;
  }
  return npy;
}

// warp-specialised step kernel: SKS_ZM_WS=1 (measured slower than the pair kernel, DESIGN.md section 11,
// profiles/r02/zws_ab_r02c.txt; kept for A/B)
static bool zm_ws() {
  static int ws = -1;
  if (ws < 0) {
    const char* e = getenv("SKS_ZM_WS");
    ws = e ? (e[0] == '1') : 0;
  }
  return ws == 1;
}

// forward-edge pair kernel (default for k <= 2 and the Chebyshev basis; SKS_ZM_FE=0 restores the two-stencil
// kernel for A/B)
static bool zm_fe() {
  static int fe = -1;
  if (fe < 0) {
    const char* e = getenv("SKS_ZM_FE");
    fe = e ? (e[0] == '1') : 1;
  }
  return fe == 1;
}

// plane-split FE kernel: thread groups per step (SKS_ZM_NG=2; default 1 = the FE pair kernel)
static int zm_ng() {
  static int ng = -1;
  if (ng < 0) {
    const char* e = getenv("SKS_ZM_NG");
    ng = e ? atoi(e) : 1;
    if (ng != 1 && ng != 2) ng = 1;
  }
  return ng;
}

template <int KM, int ZS, bool FULL, bool USL>
static cudaError_t zmp_launch(const StepArgs& a, const ZmArgs& z, const CUtensorMap& mu, const CUtensorMap& mv,
                              int grid, size_t smem, cudaStream_t st) {
  if constexpr (KM == 2) {
    // k <= 2: the next step needs <w_j, A w_j> and <w_{j-1}, A w_j> only (no window column V_l with vdot)
    if (zm_fe() && z.vdot == 0) {
      StepArgs af = a;
      af.fe = 1;
      if constexpr (ZS % 2 == 0) {
        if (zm_ng() == 2) {
          if (cudaError_t e = set_smem_attr(step3d_zfe_kernel<ZS, 2, FULL, USL>, smem)) return e;
          return launch_pdl(step3d_zfe_kernel<ZS, 2, FULL, USL>, grid, ZPT * 2, smem, st, af, z, mu, mv);
        }
      }
      const size_t smf = zm_smem_bytes_n<KM, ZS, zm_nst<KM, ZS, true>()>();
      if (cudaError_t e = set_smem_attr(step3d_zmp_kernel<KM, ZS, FULL, USL, true>, smf)) return e;
      return launch_pdl(step3d_zmp_kernel<KM, ZS, FULL, USL, true>, grid, ZPT_L, smf, st, af, z, mu, mv);
    }
  }
  if (cudaError_t e = set_smem_attr(step3d_zmp_kernel<KM, ZS, FULL, USL>, smem)) return e;
  return launch_pdl(step3d_zmp_kernel<KM, ZS, FULL, USL>, grid, ZPT_L, smem, st, a, z, mu, mv);
}

bool stencil_zm_supported(int dim, int64_t m, int k) {
  if (dim != 3 || m % 2) return false;  // TMA global strides must be multiples of 16 bytes
  const char* e = getenv("SKS_NO_ZM");
  if (e && e[0] == '1') return false;
  return zm_encode_fn();
}

// Step-balanced partition of the (tile, plane) units over the grid: a piece of len planes costs
// ceil((len + 2) / zs) steps (two halo planes), so the proportional split leaves the CTAs whose range
// crosses a column boundary up to a step behind.  Greedy fill with a cap of C steps per CTA, C the
// smallest cap that covers every unit (binary search); pieces end at column boundaries as in the kernel.
bool step_partition(int64_t units, int64_t nz, int grid, int zs, int maxg, int32_t* ub) {
  if (grid > maxg || units > INT32_MAX) return false;
  auto fill = [&](int64_t C, bool write) -> bool {
    int64_t u = 0;
    if (write) ub[0] = 0;
    for (int b = 0; b < grid; ++b) {
      int64_t k = C;
      while (u < units && k > 0) {
        const int64_t rem = nz - (u % nz);
        const int64_t cap = zs * k - 2;
        if (cap < 1) break;
        const int64_t len = std::min(rem, cap);
        u += len;
        k -= (len + 2 + zs - 1) / zs;
      }
      if (write) ub[b + 1] = (int32_t)u;
    }
    return u >= units;
  };
  int64_t lo = 1, hi = units + 2;
  while (lo < hi) {
    const int64_t mid = (lo + hi) / 2;
    if (fill(mid, false)) hi = mid;
    else lo = mid + 1;
  }
  fill(lo, true);
  return ub[grid] == units;
}

void stencil_zm_tiling(int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid) {
  a->tiles_x = (int)((m + ZX - 1) / ZX);
  a->tiles_y = (int)((m + ZY - 1) / ZY);
  a->zchunk = 0;
  a->ntiles = (int64_t)a->tiles_x * a->tiles_y * nz;  // (tile, plane) units
  *grid = (int)std::max<int64_t>(1, std::min<int64_t>(a->ntiles, (int64_t)num_sms * ZM_CPS));
}

template <int KM, bool FULL, bool USL>
static cudaError_t zm_launch_v(const StepArgs& a, const ZmArgs& z, const CUtensorMap& mu, const CUtensorMap& mv,
                               int grid, cudaStream_t st) {
  constexpr int ZS = zm_zs<KM>();
  const size_t smem = zm_smem_bytes<KM, ZS>();
  if (cudaError_t e = set_smem_attr(step3d_zm_kernel<KM, ZS, FULL, USL>, smem)) return e;
  if (zm_ws()) {
    constexpr int NST = zws_smem_bytes<KM, ZS, 3>() <= 226 * 1024 ? 3 : 2;
    constexpr size_t wsm = zws_smem_bytes<KM, ZS, NST>();
    if (cudaError_t e = set_smem_attr(step3d_zws_kernel<KM, ZS, NST, FULL, USL>, wsm)) return e;
    return launch_pdl(step3d_zws_kernel<KM, ZS, NST, FULL, USL>, grid, WS_T, wsm, st, a, z, mu, mv);
  }
  if (zm_npy() == 2) return zmp_launch<KM, ZS, FULL, USL>(a, z, mu, mv, grid, smem, st);
  return launch_pdl(step3d_zm_kernel<KM, ZS, FULL, USL>, grid, ZT, smem, st, a, z, mu, mv);
}

template <int KM>
static cudaError_t zm_launch(const StepArgs& a, const ZmArgs& z, const CUtensorMap& mu, const CUtensorMap& mv,
                             int grid, cudaStream_t st) {
  const bool full = z.nv == KM - 1;
  const bool usl = a.mode == 0 && a.k >= 2;  // step_prologue: uslot = k+1 for k >= 2 (mode 0)
  if (full && usl) return zm_launch_v<KM, true, true>(a, z, mu, mv, grid, st);
  if (full) return zm_launch_v<KM, true, false>(a, z, mu, mv, grid, st);
  if (usl) return zm_launch_v<KM, false, true>(a, z, mu, mv, grid, st);
  return zm_launch_v<KM, false, false>(a, z, mu, mv, grid, st);
}

// mode 0: U = column j-1, V_l = columns lo+l of W; mode 1: U = x, V0 = f; mode 2: U = v0.
cudaError_t launch_step_stencil_zm(const StepArgs& a, const double* W, int64_t ncol, const double* xb,
                                   const double* fb, const double* vb, int grid, cudaStream_t st, void** cache) {
  ZmMaps* mp = reinterpret_cast<ZmMaps*>(*cache);
  if (!mp) {
    mp = new ZmMaps();
    *cache = mp;
  }
  const int km = step_km(a.k);
  const int zs = km == 2 ? zm_zs<2>() : (km == 4 ? zm_zs<4>() : zm_zs<8>());
  auto upd = [&](CUtensorMap* mpp, int slot, const double* base, int64_t nc, bool ub) -> bool {
    MapKey key;
    key.base = base;
    key.ld = a.ld;
    key.nz = a.nz;
    key.m = a.m;
    key.ncol = nc;
    key.G = a.G;
    key.depth = ub ? zs + 2 : zs;
    key.kind = ub ? 1 : 0;
    if (mp->key[slot] == key) return true;
    if (!zm_encode(mpp, base, a.m, a.nz, a.G, a.ld, nc, ub, ub ? zs + 2 : zs)) return false;
    mp->key[slot] = key;
    return true;
  };
  ZmArgs z;
  memset(&z, 0, sizeof(z));
  z.tiles_x = a.tiles_x;
  z.ncolxy = a.tiles_x * a.tiles_y;
  z.units = a.ntiles;
  z.nv = (a.mode == 0) ? std::min(a.j, a.k) - 1 : (a.mode == 1 ? 1 : 0);
  z.vdot = 0;
  {
    static int sbv = -1;  // SKS_ZWS_STORE_B=1: group B stores w_j (A/B switch)
    if (sbv < 0) {
      const char* e = getenv("SKS_ZWS_STORE_B");
      sbv = e ? (e[0] == '1') : 0;
    }
    z.store_b = sbv;
  }
  if (a.mode == 0 && a.basis == 0) {  // step_prologue: vslot[l] = 3 + (lo + l) - (j - k + 1) if >= 0
    const int lo = std::max(0, a.j - a.k);
    for (int l = 0; l < z.nv; ++l)
      if (lo + l - (a.j - a.k + 1) >= 0) z.vdot |= 1 << l;
  }
  {  // step-balanced partition, cached per (units, nz, grid, zs)
    static int bal = -1;
    if (bal < 0) {
      const char* e = getenv("SKS_ZM_BALANCE");
      bal = e ? (e[0] == '1') : ZM_BALANCE_DEFAULT;
    }
    if (bal) {
      const int64_t pk = z.units * 1000003 + a.nz * 131 + grid * 7 + zs;
      if (mp->part_key != pk) {
        mp->part_ok = step_partition(z.units, a.nz, grid, zs, ZM_MAXG, mp->ub);
        mp->part_key = pk;
      }
      if (mp->part_ok) {
        z.use_ub = 1;
        memcpy(z.ub, mp->ub, sizeof(int32_t) * (grid + 1));
      }
    }
  }
  const CUtensorMap* mu;
  const CUtensorMap* mv;
  if (a.mode == 0) {
    if (!upd(&mp->WU, 0, W, ncol, true) || !upd(&mp->WV, 1, W, ncol, false)) return cudaErrorInvalidValue;
    mu = &mp->WU;
    mv = &mp->WV;
    const int lo = std::max(0, a.j - a.k);
    z.ucol = a.j - 1;
    for (int l = 0; l < a.j - 1 - lo; ++l) z.vcol[l] = lo + l;
  } else if (a.mode == 1) {
    if (!upd(&mp->XU, 2, xb, 1, true) || !upd(&mp->FV, 3, fb, 1, false)) return cudaErrorInvalidValue;
    mu = &mp->XU;
    mv = &mp->FV;
  } else {
    if (!upd(&mp->VU, 4, vb, 1, true) || !upd(&mp->WV, 1, W, ncol, false)) return cudaErrorInvalidValue;
    mu = &mp->VU;
    mv = &mp->WV;  // unused (nv = 0)
  }
  switch (km) {
    case 2: return zm_launch<2>(a, z, *mu, *mv, grid, st);
    case 4: return zm_launch<4>(a, z, *mu, *mv, grid, st);
    default: return zm_launch<8>(a, z, *mu, *mv, grid, st);
  }
}

void stencil_zm_free(void* cache) { delete reinterpret_cast<ZmMaps*>(cache); }

}  // namespace sks
