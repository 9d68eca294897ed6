// eig.cu -- the small nonsymmetric eigenproblem of sRR on the device (Alg. 2 P:1683:
// "Solve eigenvalue problem T^-1 U^* D y_i = lambda_i y_i"; "the QR algorithm").
//
//  * build_mhat: Mhat = T^-1 U^T SAB.  With a Krylov basis the paper notes Mhat and the
//    recurrence matrix "differ only in the final column":  since
//    S m_j = sum_{i<=j+1} Hbar[i,j] S b_i, and T^-1 U^T S b_i = e_i for i < d,
//        Mhat = Hbar[:d, :d] + e_{d-1}-column correction  nu_d T^-1 U^T S b_d,
//    so Mhat is upper Hessenberg by construction (no Hessenberg reduction needed).
//  * hqr: Francis double-shift QR iteration on the Hessenberg matrix, eigenvalues only
//    (one CTA; deflation and shift-origin searches over the whole block, the bulge chased by
//    one warp through 32x32 shared-memory windows, the off-window parts of each window's 29
//    reflectors applied as one accumulated-Q block update by the whole CTA).
//  * inverse iteration per selected eigenvalue on (Mhat - theta I) in complex arithmetic
//    (Hessenberg LU with partial pivoting), one CTA per eigenvalue, giving y_i.
//  * sketched residual estimate  ||D y - theta C y|| / ||C y||  (Eq. srr-resid-est).
#include <climits>
#include <cstdlib>

#include "common.cuh"
#include "internal.h"

namespace sks {

// Mhat (d x d column-major, ld = d): Hbar[:d,:d] (+ last column += t)
__global__ void build_mhat_kernel(const double* __restrict__ H, int ldH, int d, const double* __restrict__ t,
                                  const double* __restrict__ gam, double* __restrict__ Mh) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= d * d) return;
  const int i = idx % d, j = idx / d;
  double v = (i <= j + 1) ? H[i + (int64_t)j * ldH] : 0.0;
  if (j == d - 1) v += gam[d - 1] * t[i];  // A b_{d-1} = gam w_d + ...
  Mh[idx] = v;
}

#define HA(i, j) a[(i) + (int64_t)(j) * lda]

// block-wide max of an int (all threads get the result)
__device__ __forceinline__ int block_max_int(int v, int* smem) {
  for (int o = 16; o > 0; o >>= 1) v = max(v, __shfl_xor_sync(0xffffffffu, v, o));
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  __syncthreads();
  if (lane == 0) smem[wid] = v;
  __syncthreads();
  int r = lane < nw ? smem[lane] : INT_MIN;
  for (int o = 16; o > 0; o >>= 1) r = max(r, __shfl_xor_sync(0xffffffffu, r, o));
  return r;
}

// 1/x and 1/sqrt(x) from the hardware approximations plus two Newton steps each (about 1 ulp;
// used for reflector coefficients, where the IEEE-exact slow paths only add latency)
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  double e = fma(-x, y, 1.0);
  y = fma(y, e, y);
  e = fma(-x, y, 1.0);
  return fma(y, e, y);
}
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// D(8x8) += A(8x4, row) B(4x8, col) in fp64 on the tensor cores; per thread: a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], d0/d1 = D[lane/4][2(lane%4)], D[lane/4][2(lane%4)+1]
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// reflector of (p, q, r) in the form of the Francis sweep: s = sign(p) ||(p,q,r)||,
// u = (p+s, q, r)/s, w = (1, q/(p+s), r/(p+s)), P = I - u w^T; (p,q,r) = 0 gives u = 0 (P = I)
struct HqRefl {
  double xx, yy, zz, qq, rr, s;
  bool valid;
};
__device__ __forceinline__ HqRefl hq_refl(double p, double q, double r) {
  HqRefl R;
  const double t = fma(p, p, fma(q, q, r * r));
  double s, is;
  if (t > 1e-280 && t < 1e280) {
    is = rsqrt_nr(t);
    s = t * is;
  } else {
    const double x = fabs(p) + fabs(q) + fabs(r);
    if (x == 0.0) {
      R.xx = R.yy = R.zz = R.qq = R.rr = R.s = 0.0;
      R.valid = false;
      return R;
    }
    const double ix = 1.0 / x, ps = p * ix, qs = q * ix, rs = r * ix;
    s = x * sqrt(ps * ps + qs * qs + rs * rs);
    is = 1.0 / s;
  }
  if (p < 0.0) {
    s = -s;
    is = -is;
  }
  const double pp = p + s, ip = rcp_nr(pp);
  R.s = s;
  R.xx = pp * is;
  R.yy = q * is;
  R.zz = r * is;
  R.qq = q * ip;
  R.rr = r * ip;
  R.valid = true;
  return R;
}

// branch-free variant for the chase (the matrix is pre-scaled to norm ~1, so p^2+q^2+r^2 cannot
// overflow; a sub-normal-range bulge is treated as zero, i.e. P = I)
__device__ __forceinline__ HqRefl hq_identity() {  // P = I (no arithmetic)
  HqRefl R;
  R.xx = R.yy = R.zz = R.qq = R.rr = R.s = 0.0;
  R.valid = false;
  return R;
}
__device__ __forceinline__ HqRefl hq_refl_fast(double p, double q, double r) {
  HqRefl R;
  const double t = fma(p, p, fma(q, q, r * r));
  const bool ok = t >= 2.3e-308;
  double is = rsqrt_nr(ok ? t : 1.0);
  double s = t * is;
  s = p < 0.0 ? -s : s;
  is = p < 0.0 ? -is : is;
  const double pp = p + s, ip = rcp_nr(ok ? pp : 1.0);
  R.s = s;
  R.xx = ok ? pp * is : 0.0;
  R.yy = ok ? q * is : 0.0;
  R.zz = ok ? r * is : 0.0;
  R.qq = ok ? q * ip : 0.0;
  R.rr = ok ? r * ip : 0.0;
  R.valid = ok;
  return R;
}

// Short-chain reflector (HQ_NEWNR, default): third-order refinements of 1/sqrt(t) and 1/(p+s) (one correction
// each instead of two Newton steps) and the seed of 1/(p+s) formed from the approximate root off the dependent
// chain: C5 chase 44.5M -> 40.1M cycles (tools/ab_hqr.sh, profiles/r02/hqr_ab_r02.txt).  is = 1/s and
// ip = 1/(p+s) are kept for hq_next_x (HQ_FASTX=1: the next bulge input in two operations after 1/(p+s) instead
// of seven; measured slower, 43.8M cycles -- more instructions per round, so the round is not bound by this chain)
#ifndef HQ_FASTX
#define HQ_FASTX 0
#endif
#ifndef HQ_NEWNR
#define HQ_NEWNR 1
#endif
// HQ_XPF (default, HQ_NB == 3): window transitions without L2 round trips on the critical path -- while the
// chase runs, the spare warps write the previous window back, apply its deferred off-window update and then
// prefetch what the next window needs from global memory (the rows below this window into the second window
// buffer, this window's rows x the next window's new columns into Xb); after the chase the next window is
// assembled in shared memory (overlap copy + Q^T Xb) and the chase resumes
#ifndef HQ_XPF
#define HQ_XPF 1
#endif
struct HqRefl2 {
  HqRefl R;
  double is, ip;
};
__device__ __forceinline__ HqRefl2 hq_refl_fast2(double p, double q, double r) {
  HqRefl2 O;
  const double t = fma(p, p, fma(q, q, r * r));
  const bool ok = t >= 2.3e-308;
  const double tt = ok ? t : 1.0;
  double ya;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(ya) : "d"(tt));
  const double sa = tt * ya;
  double ipa;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(ipa) : "d"(p + (p < 0.0 ? -sa : sa)));
#if HQ_NEWNR
  const double e = fma(-tt * ya, ya, 1.0);
  double is = fma(ya * e, fma(e, 0.375, 0.5), ya);  // ya (1 + e/2 + 3e^2/8)
#else
  double is = rsqrt_nr(tt);
#endif
  double s = tt * is;
  s = p < 0.0 ? -s : s;
  is = p < 0.0 ? -is : is;
  const double pp = p + s;
#if HQ_NEWNR
  const double e2 = fma(-pp, ipa, 1.0);
  const double ip = fma(ipa * e2, 1.0 + e2, ipa);  // ipa (1 + e2 + e2^2)
#else
  const double ip = rcp_nr(ok ? pp : 1.0);
  (void)ipa;
#endif
  O.R.s = s;
  O.R.xx = ok ? pp * is : 0.0;
  O.R.yy = ok ? q * is : 0.0;
  O.R.zz = ok ? r * is : 0.0;
  O.R.qq = ok ? q * ip : 0.0;
  O.R.rr = ok ? r * ip : 0.0;
  O.R.valid = ok;
  O.is = ok ? is : 0.0;
  O.ip = ok ? ip : 0.0;
  return O;
}
// The next bulge input H[k+1..k+3][k] after step k's two-sided transformation, from the step's input x = (p, q, r)
// and the 3x3 block B = H[k..k+2][k..k+2] before the step.  With u = (p+s, q, r)/s, 1 - u_0 = -p/s, so
//   N_i0 = (1-u_0) R_i0 - u_1 R_i1 - u_2 R_i2 = -is (x.B_i) + u_i is (x.B_0 + ip (q x.B_1 + r x.B_2))   (i = 1, 2)
//   N_30 = -u_2 h3,
// where x.B_i = p B_i0 + q B_i1 + r B_i2 need no reflector quantity: only two operations follow 1/(p+s) on the
// dependent chain (the explicit form needs seven).  Same values up to rounding (validated: max 7e-16 relative).
__device__ __forceinline__ void hq_next_x(const HqRefl2& R, double p, double q, double r, double B00, double B01,
                                          double B02, double B10, double B11, double B12, double B20, double B21,
                                          double B22, double h3, double& np, double& nq, double& nr) {
  const double xB0 = fma(r, B02, fma(q, B01, p * B00));
  const double xB1 = fma(r, B12, fma(q, B11, p * B10));
  const double xB2 = fma(r, B22, fma(q, B21, p * B20));
  const double xQ = fma(r, xB2, q * xB1);
  const double a1 = -R.is * xB1, a2 = -R.is * xB2, v1 = R.R.yy * R.is, v2 = R.R.zz * R.is;
  const double g = fma(R.ip, xQ, xB0);
  np = R.R.valid ? fma(v1, g, a1) : B10;
  nq = R.R.valid ? fma(v2, g, a2) : B20;
  nr = -R.R.zz * h3;
}

// per-lane scratch of the masked stores: HQ_SS doubles per lane (odd: the lanes of a half-warp hit distinct banks;
// 16 made every masked access a 16-way bank conflict -- ncu: 16.4M conflicts per C5 launch)
#ifndef HQ_SS
#define HQ_SS 17
#endif
constexpr int HQ_R = 32;         // window rows/cols (the bulge region of HQ_W steps plus 3)
constexpr int HQ_W = HQ_R - 3;   // bulge steps per window
constexpr int HQ_LD = HQ_R + 1;  // odd pitch: row- and column-wise smem access both conflict-free
#ifndef HQ_NB
// bulges per Francis sweep / chasing warps:
//   1: one bulge, one warp (hqr 29 ms at C5, 422 sweeps);
//   2: two bulges with the same shift pair chased by ONE warp (hq_chase2; 269 sweeps but the warp
//      issues both chains: 40 ms);
//   3: the same two bulges on two warps with a 64-thread barrier per round (hq_chase2w; 27 ms).
#define HQ_NB 3
#endif
constexpr int HQ_THREADS = HQ_NB == 2 ? 256 : 384;  // (HQ_NB=3: warps 0, 1 chase)  // HQ_NB=2 needs the larger register budget
constexpr int HQ_QSZ = HQ_LD * HQ_R;
#ifndef HQ_TWO_MIN
#define HQ_TWO_MIN 12  // minimum nn - m per additional bulge
#endif
#ifndef HQ_NW
#define HQ_NW 2  // HQ_NB=3: chase warps (bulges per sweep)
#endif

// ---- two-bulge chase (HQ_NB == 2): bulges A (leading) and B (trailing by 4 positions) carry the same
// double shift (reading: two Francis double-shift steps with one shift pair per sweep; B is introduced
// at row m from the current matrix once A has moved 4 positions).  P_A (rows/cols kA..kA+2) and P_B
// (kB..kB+2, kB = kA-4) act on disjoint index sets, so each round applies both in one shared-memory
// phase: the block rows kB..kB+2 x cols kA..kA+2 (touched by P_B from the left and P_A from the right)
// is formed by the lanes of A's column transform.  The two reflector chains are independent, so the
// scheduler overlaps their FP64 latencies.  Window: rows/cols [lo, lo+31] (col lo-1 for reflector
// reads), rounds kA in [a0, a1); Q accumulates P_A and P_B.
struct HqBulge {
  double B00, B01, B02, B10, B11, B12, B20, B21, B22;  // H[k..k+2][k..k+2] before the step
  double C0, C1, C2, h3, d33;                         // H[k..k+2][k+3], H[k+3][k+2], H[k+3][k+3]
};

// ---- two-bulge chase on two warps (HQ_NB == 3): warp 0 chases bulge A, warp 1 bulge B (4 rows
// behind, same shift pair), one 64-thread named barrier per round.  Within a round the two warps
// touch disjoint entries: the block rows kB..kB+2 x cols kA..kA+2 is formed by warp 0 (P_B from the
// left with B's reflector of the round, exchanged through shared memory one round ahead, then P_A);
// B's row transformation skips those columns; B reloads its column kB+3 and row kB+3 every round
// (A changes them).  Validated against tools/micro/hq_kern2.py (same arithmetic as hq_chase2).
__device__ __forceinline__ void hq_bar2() { asm volatile("bar.sync 1, 64;" ::: "memory"); }

__device__ __forceinline__ void hq_chase2w(double* Hw, double* Qs, double* dmy, double* xchg, int lo, int r1, int a0,
                                           int a1, int m, int nn, int l, double sp, double sq, double sr, double sx,
                                           double sy, double sw, int lane, int role) {
  auto H_ = [&](int gi, int gj) -> double {
    return (gi >= lo && gj >= lo - 1 && gi <= r1 && gj <= r1) ? Hw[(gi - lo) + (gj - lo + 1) * HQ_LD] : 0.0;
  };
  auto load_state = [&](int k, HqBulge& S) {
    S.B00 = H_(k, k); S.B01 = H_(k, k + 1); S.B02 = H_(k, k + 2);
    S.B10 = H_(k + 1, k); S.B11 = H_(k + 1, k + 1); S.B12 = H_(k + 1, k + 2);
    S.B20 = H_(k + 2, k); S.B21 = H_(k + 2, k + 1); S.B22 = H_(k + 2, k + 2);
    S.C0 = H_(k, k + 3); S.C1 = H_(k + 1, k + 3); S.C2 = H_(k + 2, k + 3);
    S.h3 = H_(k + 3, k + 2); S.d33 = H_(k + 3, k + 3);
  };
  auto put = [&](const HqRefl& R, int slot) {  // B's reflector for warp 0
    if (lane == 0) {
      double* x = xchg + 8 * slot;
      x[0] = R.xx; x[1] = R.yy; x[2] = R.zz; x[3] = R.qq; x[4] = R.rr; x[5] = R.s; x[6] = R.valid ? 1.0 : 0.0;
    }
  };
  auto get = [&](int slot) {
    const double* x = xchg + 8 * slot;
    HqRefl R;
    R.xx = x[0]; R.yy = x[1]; R.zz = x[2]; R.qq = x[3]; R.rr = x[4]; R.s = x[5]; R.valid = x[6] != 0.0;
    return R;
  };
  const bool twoB = nn - m >= HQ_TWO_MIN;
  HqBulge S = {};
  HqRefl2 RX = hq_refl_fast2(0.0, 0.0, 0.0);
  HqRefl& R = RX.R;
  double xp = 0.0, xq = 0.0, xr = 0.0;  // this warp's current reflector input
  // ---- window start: each warp its own bulge
  if (role == 0) {
    const int kA = a0;
    if (kA <= nn - 1) {
      double p, q, r;
      if (kA == m) {
        p = sp; q = sq; r = sr;
      } else {
        p = H_(kA, kA - 1); q = H_(kA + 1, kA - 1); r = H_(kA + 2, kA - 1);
      }
      load_state(kA, S);
      RX = hq_refl_fast2(p, q, r);
      xp = p; xq = q; xr = r;
    }
  } else {
    const int kB = a0 - 4;
    if (twoB && kB >= m && kB <= nn - 1) {
      load_state(kB, S);
      xp = H_(kB, kB - 1); xq = H_(kB + 1, kB - 1); xr = H_(kB + 2, kB - 1);
      RX = hq_refl_fast2(xp, xq, xr);
    } else if (twoB && kB + 1 == m) {  // B enters at the window's first round
      // (cannot happen: B enters at kA = m+4 inside the sweep's first window)
    }
    put(R, a0 & 1);
  }
  hq_bar2();
  for (int kA = a0; kA < a1; ++kA) {
    const int kB = kA - 4;
    const bool actA = kA <= nn - 1, actB = twoB && kB >= m && kB <= nn - 1;
    const int ir = lo + lane;
    if (role == 0) {
      const HqRefl RB = get(kA & 1);  // B's reflector of this round (identity if B is not running)
      const double v0 = RB.xx, v1 = RB.yy, v2 = RB.zz, x1 = RB.qq, x2 = RB.rr;
      double E0, E1, E2, E3, h4, d44;
      double Z[3][3];
      {
        E0 = H_(kA, kA + 4); E1 = H_(kA + 1, kA + 4); E2 = H_(kA + 2, kA + 4); E3 = H_(kA + 3, kA + 4);
        h4 = H_(kA + 4, kA + 3); d44 = H_(kA + 4, kA + 4);
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) Z[i][j] = H_(kB + i, kA + j);
      }
      const int jA = kA + 3 + lane;
      const bool rokA = actA && jA <= r1;
      double* colA = rokA ? Hw + (jA - lo + 1) * HQ_LD + (kA - lo) : dmy + HQ_SS * lane;
      const double aA0 = colA[0], aA1 = colA[1], aA2 = colA[2];
      const bool cokA = actA && ir <= min(nn, kA + 3);
      const bool specA = ir >= kB && ir <= kB + 2;
      const bool ldA = cokA && ir < kA && !specA;
      double* rowA = Hw + lane + (kA - lo + 1) * HQ_LD;
      const double bA0 = ldA ? rowA[0] : 0.0, bA1 = ldA ? rowA[HQ_LD] : 0.0, bA2 = ldA ? rowA[2 * HQ_LD] : 0.0;
      double* qA = Qs + lane + (actA ? kA - lo : 0) * HQ_LD;
      const double gA0 = qA[0], gA1 = qA[HQ_LD], gA2 = qA[2 * HQ_LD];
      double* hkA = (lane == 0 && actA && R.valid) ? Hw + (kA - lo) + (kA - lo) * HQ_LD : dmy + HQ_SS * lane + 6;
      const double hkAv = *hkA;
      const double u0 = R.xx, u1 = R.yy, u2 = R.zz, w1 = R.qq, w2 = R.rr;
      const double pp0 = fma(w2, S.B20, fma(w1, S.B10, S.B00)), pp1 = fma(w2, S.B21, fma(w1, S.B11, S.B01)),
                   pp2 = fma(w2, S.B22, fma(w1, S.B12, S.B02)), ppc = fma(w2, S.C2, fma(w1, S.C1, S.C0)),
                   ppe = fma(w2, E2, fma(w1, E1, E0));
      const double R10 = fma(-u1, pp0, S.B10), R11 = fma(-u1, pp1, S.B11), R12 = fma(-u1, pp2, S.B12),
                   R1c = fma(-u1, ppc, S.C1), R1e = fma(-u1, ppe, E1);
      const double R20 = fma(-u2, pp0, S.B20), R21 = fma(-u2, pp1, S.B21), R22 = fma(-u2, pp2, S.B22),
                   R2c = fma(-u2, ppc, S.C2), R2e = fma(-u2, ppe, E2);
      const double t1 = fma(u2, R12, fma(u1, R11, u0 * R10));
      const double t2 = fma(u2, R22, fma(u1, R21, u0 * R20));
      const double t3 = u2 * S.h3;
      const double N10 = R10 - t1, N11 = fma(-t1, w1, R11), N12 = fma(-t1, w2, R12);
      const double N20 = R20 - t2, N21 = fma(-t2, w1, R21), N22 = fma(-t2, w2, R22);
      const double N30 = -t3, N31 = -t3 * w1, N32 = fma(-t3, w2, S.h3);
      const bool nx = actA && kA + 1 <= nn - 1;
#if HQ_FASTX
      double np_, nq_, nr_;
      hq_next_x(RX, xp, xq, xr, S.B00, S.B01, S.B02, S.B10, S.B11, S.B12, S.B20, S.B21, S.B22, S.h3, np_, nq_, nr_);
      np_ = nx ? np_ : 0.0; nq_ = nx ? nq_ : 0.0; nr_ = nx ? nr_ : 0.0;
      (void)N10; (void)N20; (void)N30;
      const HqRefl2 RnX = hq_refl_fast2(np_, nq_, nr_);
#else
      const HqRefl2 RnX = hq_refl_fast2(nx ? N10 : 0.0, nx ? N20 : 0.0, nx ? N30 : 0.0);
      const double np_ = nx ? N10 : 0.0, nq_ = nx ? N20 : 0.0, nr_ = nx ? N30 : 0.0;
#endif
      *hkA = (kA == m) ? ((l != m) ? -hkAv : hkAv) : -R.s;
      {
        const double pr = fma(w2, aA2, fma(w1, aA1, aA0));
        colA[0] = fma(-u0, pr, aA0);
        colA[1] = fma(-u1, pr, aA1);
        *((rokA && kA + 2 <= nn) ? colA + 2 : dmy + HQ_SS * lane + 2) = fma(-u2, pr, aA2);
      }
      {
        const int d = ir - kA, dB = ir - kB;
        const double X0 = fma(-u0, pp0, S.B00), X1 = fma(-u0, pp1, S.B01), X2 = fma(-u0, pp2, S.B02);
        const double zz0 = fma(x2, Z[2][0], fma(x1, Z[1][0], Z[0][0]));
        const double zz1 = fma(x2, Z[2][1], fma(x1, Z[1][1], Z[0][1]));
        const double zz2 = fma(x2, Z[2][2], fma(x1, Z[1][2], Z[0][2]));
        const double vb = dB == 0 ? v0 : (dB == 1 ? v1 : v2);
        const double zr0 = fma(-vb, zz0, dB == 0 ? Z[0][0] : (dB == 1 ? Z[1][0] : Z[2][0]));
        const double zr1 = fma(-vb, zz1, dB == 0 ? Z[0][1] : (dB == 1 ? Z[1][1] : Z[2][1]));
        const double zr2 = fma(-vb, zz2, dB == 0 ? Z[0][2] : (dB == 1 ? Z[1][2] : Z[2][2]));
        const bool own = ir >= kA;
        const double c0 = specA ? zr0 : (own ? (d == 0 ? X0 : (d == 1 ? R10 : (d == 2 ? R20 : 0.0))) : bA0);
        const double c1 = specA ? zr1 : (own ? (d == 0 ? X1 : (d == 1 ? R11 : (d == 2 ? R21 : 0.0))) : bA1);
        const double c2 = specA ? zr2 : (own ? (d == 0 ? X2 : (d == 1 ? R12 : (d == 2 ? R22 : S.h3))) : bA2);
        const double tt = fma(u2, c2, fma(u1, c1, u0 * c0));
        double* sc = dmy + HQ_SS * lane;
        *(cokA ? rowA : sc) = c0 - tt;
        *(cokA && kA + 1 <= nn ? rowA + HQ_LD : sc + 1) = fma(-tt, w1, c1);
        *(cokA && kA + 2 <= nn ? rowA + 2 * HQ_LD : sc + 2) = fma(-tt, w2, c2);
      }
      {
        double* sq2 = dmy + HQ_SS * lane + 8;
        const double tq = fma(u2, gA2, fma(u1, gA1, u0 * gA0));
        *(actA ? qA : sq2) = gA0 - tq;
        *(actA ? qA + HQ_LD : sq2 + 1) = fma(-tq, w1, gA1);
        *(actA ? qA + 2 * HQ_LD : sq2 + 2) = fma(-tq, w2, gA2);
      }
      RX = RnX;
      xp = np_; xq = nq_; xr = nr_;
      S.B00 = N11; S.B01 = N12; S.B02 = R1c;
      S.B10 = N21; S.B11 = N22; S.B12 = R2c;
      S.B20 = N31; S.B21 = N32; S.B22 = S.d33;
      S.C0 = R1e; S.C1 = R2e; S.C2 = E3;
      S.h3 = h4; S.d33 = d44;
    } else {
      HqRefl2 RnextX = hq_refl_fast2(0.0, 0.0, 0.0);
      double np_ = 0.0, nq_ = 0.0, nr_ = 0.0;
      if (actB) {
        {
          S.C0 = H_(kB, kB + 3); S.C1 = H_(kB + 1, kB + 3); S.C2 = H_(kB + 2, kB + 3);
          S.h3 = H_(kB + 3, kB + 2); S.d33 = H_(kB + 3, kB + 3);
        }
        const int jB = kB + 3 + lane;
        const bool rokB = jB <= r1 && (!actA || lane < 1 || lane > 3);
        double* colB = rokB ? Hw + (jB - lo + 1) * HQ_LD + (kB - lo) : dmy + HQ_SS * lane + 3;
        const double aB0 = colB[0], aB1 = colB[1], aB2 = colB[2];
        const bool cokB = ir <= min(nn, kB + 3);
        const bool ldB = cokB && ir < kB;
        double* rowB = Hw + lane + (kB - lo + 1) * HQ_LD;
        const double bB0 = ldB ? rowB[0] : 0.0, bB1 = ldB ? rowB[HQ_LD] : 0.0, bB2 = ldB ? rowB[2 * HQ_LD] : 0.0;
        double* qB = Qs + lane + (kB - lo) * HQ_LD;
        const double gB0 = qB[0], gB1 = qB[HQ_LD], gB2 = qB[2 * HQ_LD];
        double* hkB = (lane == 0 && R.valid) ? Hw + (kB - lo) + (kB - lo) * HQ_LD : dmy + HQ_SS * lane + 7;
        const double hkBv = *hkB;
        const double v0 = R.xx, v1 = R.yy, v2 = R.zz, x1 = R.qq, x2 = R.rr;
        const double qq0 = fma(x2, S.B20, fma(x1, S.B10, S.B00)), qq1 = fma(x2, S.B21, fma(x1, S.B11, S.B01)),
                     qq2 = fma(x2, S.B22, fma(x1, S.B12, S.B02)), qqc = fma(x2, S.C2, fma(x1, S.C1, S.C0));
        const double S10 = fma(-v1, qq0, S.B10), S11 = fma(-v1, qq1, S.B11), S12 = fma(-v1, qq2, S.B12),
                     S1c = fma(-v1, qqc, S.C1);
        const double S20 = fma(-v2, qq0, S.B20), S21 = fma(-v2, qq1, S.B21), S22 = fma(-v2, qq2, S.B22),
                     S2c = fma(-v2, qqc, S.C2);
        const double e1 = fma(v2, S12, fma(v1, S11, v0 * S10));
        const double e2 = fma(v2, S22, fma(v1, S21, v0 * S20));
        const double e3 = v2 * S.h3;
        const double M10 = S10 - e1, M11 = fma(-e1, x1, S11), M12 = fma(-e1, x2, S12);
        const double M20 = S20 - e2, M21 = fma(-e2, x1, S21), M22 = fma(-e2, x2, S22);
        const double M30 = -e3, M31 = -e3 * x1, M32 = fma(-e3, x2, S.h3);
        const bool nx = kB + 1 <= nn - 1;
#if HQ_FASTX
        hq_next_x(RX, xp, xq, xr, S.B00, S.B01, S.B02, S.B10, S.B11, S.B12, S.B20, S.B21, S.B22, S.h3, np_, nq_,
                  nr_);
        np_ = nx ? np_ : 0.0; nq_ = nx ? nq_ : 0.0; nr_ = nx ? nr_ : 0.0;
        (void)M10; (void)M20; (void)M30;
#else
        np_ = nx ? M10 : 0.0; nq_ = nx ? M20 : 0.0; nr_ = nx ? M30 : 0.0;
#endif
        RnextX = hq_refl_fast2(np_, nq_, nr_);
        *hkB = (kB == m) ? ((l != m) ? -hkBv : hkBv) : -R.s;
        {
          const double pr = fma(x2, aB2, fma(x1, aB1, aB0));
          colB[0] = fma(-v0, pr, aB0);
          colB[1] = fma(-v1, pr, aB1);
          *((rokB && kB + 2 <= nn) ? colB + 2 : dmy + HQ_SS * lane + 5) = fma(-v2, pr, aB2);
        }
        {
          const int d = ir - kB;
          const double Y0 = fma(-v0, qq0, S.B00), Y1 = fma(-v0, qq1, S.B01), Y2 = fma(-v0, qq2, S.B02);
          const bool own = ir >= kB;
          const double c0 = own ? (d == 0 ? Y0 : (d == 1 ? S10 : (d == 2 ? S20 : 0.0))) : bB0;
          const double c1 = own ? (d == 0 ? Y1 : (d == 1 ? S11 : (d == 2 ? S21 : 0.0))) : bB1;
          const double c2 = own ? (d == 0 ? Y2 : (d == 1 ? S12 : (d == 2 ? S22 : S.h3))) : bB2;
          const double tt = fma(v2, c2, fma(v1, c1, v0 * c0));
          double* sc = dmy + HQ_SS * lane + 3;
          *(cokB ? rowB : sc) = c0 - tt;
          *(cokB ? rowB + HQ_LD : sc + 1) = fma(-tt, x1, c1);
          *((cokB && kB + 2 <= nn) ? rowB + 2 * HQ_LD : sc + 2) = fma(-tt, x2, c2);
        }
        {
          const double tq = fma(v2, gB2, fma(v1, gB1, v0 * gB0));
          qB[0] = gB0 - tq;
          qB[HQ_LD] = fma(-tq, x1, gB1);
          qB[2 * HQ_LD] = fma(-tq, x2, gB2);
        }
        S.B00 = M11; S.B01 = M12; S.B02 = S1c;
        S.B10 = M21; S.B11 = M22; S.B12 = S2c;
        S.B20 = M31; S.B21 = M32; S.B22 = S.d33;
      }
      if (twoB && kB + 1 == m) {  // B enters next round: its first reflector from the current matrix
        // (rows/cols m..m+2 are final: A is at m+3 and only touches indices >= m+3)
        const double z = H_(m, m), rr = sx - z, ss = sy - z;
        const double p = (rr * ss - sw) / H_(m + 1, m) + H_(m, m + 1);
        const double q = H_(m + 1, m + 1) - z - rr - ss;
        const double r = H_(m + 2, m + 1);
        load_state(m, S);
        S.B20 = 0.0;  // H[m+2][m]: zeroed by A's step m+1 (shared memory holds A's stale bulge entry)
        RnextX = hq_refl_fast2(p, q, r);
        np_ = p; nq_ = q; nr_ = r;
      }
      RX = RnextX;
      xp = np_; xq = nq_; xr = nr_;
      put(R, (kA + 1) & 1);
    }
    hq_bar2();
  }
}

// ---- NW bulges on NW warps (HQ_NB == 3; HQ_NW = 2 is the two-bulge chase above, generalised): warp w
// chases bulge w at k_w = kA - 4w with the sweep's shift pair.  Per round, warp w (a) skips the columns
// k_{w-1}..k_{w-1}+2 of the bulge ahead in its row transformation, (b) forms the block rows
// k_{w+1}..k_{w+1}+2 x its columns (P_{w+1} from the left with the reflector warp w+1 published one
// round ahead, then its own P_w), (c) reloads its column k_w+3 and row k_w+3 every round when a bulge
// runs ahead (warp 0 forwards them in registers).  Bulge w enters at row m once bulge w-1 has moved
// 4 rows; blocks too short for it (nn - m < HQ_TWO_MIN w) run fewer bulges.
__device__ __forceinline__ int hq_nbulges(int nn, int m) {
  int nb = 1;
  while (nb < HQ_NW && nn - m >= HQ_TWO_MIN * nb) ++nb;
  return nb;
}

__device__ __forceinline__ void hq_barw(int nw) { asm volatile("bar.sync 1, %0;" ::"r"(32 * nw) : "memory"); }

__device__ __forceinline__ void hq_chasew(double* Hw, double* Qs, double* dmy, double* xchg, int lo, int r1, int a0,
                                          int a1, int m, int nn, int l, double sp, double sq, double sr, double sx,
                                          double sy, double sw, int lane, int w) {
  auto H_ = [&](int gi, int gj) -> double {
    return (gi >= lo && gj >= lo - 1 && gi <= r1 && gj <= r1) ? Hw[(gi - lo) + (gj - lo + 1) * HQ_LD] : 0.0;
  };
  auto load_state = [&](int k, HqBulge& S) {
    S.B00 = H_(k, k); S.B01 = H_(k, k + 1); S.B02 = H_(k, k + 2);
    S.B10 = H_(k + 1, k); S.B11 = H_(k + 1, k + 1); S.B12 = H_(k + 1, k + 2);
    S.B20 = H_(k + 2, k); S.B21 = H_(k + 2, k + 1); S.B22 = H_(k + 2, k + 2);
    S.C0 = H_(k, k + 3); S.C1 = H_(k + 1, k + 3); S.C2 = H_(k + 2, k + 3);
    S.h3 = H_(k + 3, k + 2); S.d33 = H_(k + 3, k + 3);
  };
  auto put = [&](const HqRefl& R, int slot) {  // warp w's reflector, for warp w-1
    if (lane == 0) {
      double* x = xchg + 16 * w + 8 * slot;
      x[0] = R.xx; x[1] = R.yy; x[2] = R.zz; x[3] = R.qq; x[4] = R.rr; x[5] = R.s; x[6] = R.valid ? 1.0 : 0.0;
    }
  };
  auto get = [&](int ww, int slot) {
    const double* x = xchg + 16 * ww + 8 * slot;
    HqRefl R;
    R.xx = x[0]; R.yy = x[1]; R.zz = x[2]; R.qq = x[3]; R.rr = x[4]; R.s = x[5]; R.valid = x[6] != 0.0;
    return R;
  };
  const int nb = hq_nbulges(nn, m);
  const int NWc = HQ_NW;                 // warps in the barrier (all chase warps take part)
  const bool en = w < nb;                // this warp's bulge runs in this sweep
  HqBulge S = {};
  HqRefl R = hq_identity();
  {  // window start
    const int k = a0 - 4 * w;
    if (en && k >= m && k <= nn - 1) {
      double p, q, r;
      if (k == m) {
        p = sp; q = sq; r = sr;  // (only bulge 0 can start a window at m)
      } else {
        p = H_(k, k - 1); q = H_(k + 1, k - 1); r = H_(k + 2, k - 1);
      }
      load_state(k, S);
      R = hq_refl_fast(p, q, r);
    }
    if (w > 0) put(R, a0 & 1);
  }
  hq_barw(NWc);
  for (int kA = a0; kA < a1; ++kA) {
    const int k = kA - 4 * w;
    const bool act = en && k >= m && k <= nn - 1;
    HqRefl Rn = hq_identity();
    if (act) {
      auto cok_pre = [&](int r) { return r <= min(nn, k + 3); };
      const int ir = lo + lane;
      // rows of a bulge behind (u = w + jb, rows k_u..k_u+2, k_u = k - 4 jb) x own columns: P_u from the
      // left (its reflector, published one round ahead) before this warp's P_w
      const int off = k - ir, jb = (off + 3) >> 2, tb = 4 * jb - off;
      const bool spec = cok_pre(ir) && off >= 2 && tb <= 2 && w + jb < nb;
      const HqRefl RB = spec ? get(w + jb, kA & 1) : hq_identity();
      const double v0 = RB.xx, v1 = RB.yy, v2 = RB.zz, x1 = RB.qq, x2 = RB.rr;
      const int kb_l = k - 4 * jb;  // this lane's behind-bulge row origin
      if (w > 0) {  // column k+3 and row k+3 change under the bulge ahead: reload
        S.C0 = H_(k, k + 3); S.C1 = H_(k + 1, k + 3); S.C2 = H_(k + 2, k + 3);
        S.h3 = H_(k + 3, k + 2); S.d33 = H_(k + 3, k + 3);
      }
      const double E0 = H_(k, k + 4), E1 = H_(k + 1, k + 4), E2 = H_(k + 2, k + 4), E3 = H_(k + 3, k + 4);
      const double h4 = H_(k + 4, k + 3), d44 = H_(k + 4, k + 4);
      double Z[3][3];  // this lane's behind-bulge rows x own columns
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) Z[i][j] = spec ? H_(kb_l + i, k + j) : 0.0;
      // row transformation column k+3+lane; the columns of a running bulge ahead (v = w - ja,
      // cols k_v..k_v+2, k_v = k + 4 ja <= nn-1) are formed by that bulge's warp
      const int jc = k + 3 + lane, dc = jc - k, ja = dc >> 2, ta = dc & 3;
      const bool skip = ja >= 1 && ta <= 2 && w - ja >= 0 && k + 4 * ja <= nn - 1;
      const bool rok = jc <= r1 && !skip;
      double* colp = rok ? Hw + (jc - lo + 1) * HQ_LD + (k - lo) : dmy + HQ_SS * lane;
      const double aa0 = colp[0], aa1 = colp[1], aa2 = colp[2];
      const bool cok = cok_pre(ir);
      const bool ld = cok && ir < k && !spec;
      double* rowp = Hw + lane + (k - lo + 1) * HQ_LD;
      const double b0 = ld ? rowp[0] : 0.0, b1 = ld ? rowp[HQ_LD] : 0.0, b2 = ld ? rowp[2 * HQ_LD] : 0.0;
      double* qp = Qs + lane + (k - lo) * HQ_LD;
      const double g0 = qp[0], g1 = qp[HQ_LD], g2 = qp[2 * HQ_LD];
      double* hk = (lane == 0 && R.valid) ? Hw + (k - lo) + (k - lo) * HQ_LD : dmy + HQ_SS * lane + 6;
      const double hkv = *hk;
      const double u0 = R.xx, u1 = R.yy, u2 = R.zz, w1 = R.qq, w2 = R.rr;
      const double pp0 = fma(w2, S.B20, fma(w1, S.B10, S.B00)), pp1 = fma(w2, S.B21, fma(w1, S.B11, S.B01)),
                   pp2 = fma(w2, S.B22, fma(w1, S.B12, S.B02)), ppc = fma(w2, S.C2, fma(w1, S.C1, S.C0)),
                   ppe = fma(w2, E2, fma(w1, E1, E0));
      const double R10 = fma(-u1, pp0, S.B10), R11 = fma(-u1, pp1, S.B11), R12 = fma(-u1, pp2, S.B12),
                   R1c = fma(-u1, ppc, S.C1), R1e = fma(-u1, ppe, E1);
      const double R20 = fma(-u2, pp0, S.B20), R21 = fma(-u2, pp1, S.B21), R22 = fma(-u2, pp2, S.B22),
                   R2c = fma(-u2, ppc, S.C2), R2e = fma(-u2, ppe, E2);
      const double t1 = fma(u2, R12, fma(u1, R11, u0 * R10));
      const double t2 = fma(u2, R22, fma(u1, R21, u0 * R20));
      const double t3 = u2 * S.h3;
      const double N10 = R10 - t1, N11 = fma(-t1, w1, R11), N12 = fma(-t1, w2, R12);
      const double N20 = R20 - t2, N21 = fma(-t2, w1, R21), N22 = fma(-t2, w2, R22);
      const double N30 = -t3, N31 = -t3 * w1, N32 = fma(-t3, w2, S.h3);
      const bool nx = k + 1 <= nn - 1;
      Rn = hq_refl_fast(nx ? N10 : 0.0, nx ? N20 : 0.0, nx ? N30 : 0.0);
      *hk = (k == m) ? ((l != m) ? -hkv : hkv) : -R.s;
      {
        const double pr = fma(w2, aa2, fma(w1, aa1, aa0));
        colp[0] = fma(-u0, pr, aa0);
        colp[1] = fma(-u1, pr, aa1);
        *((rok && k + 2 <= nn) ? colp + 2 : dmy + HQ_SS * lane + 2) = fma(-u2, pr, aa2);
      }
      {
        const int d = ir - k, dB = tb;
        const double X0 = fma(-u0, pp0, S.B00), X1 = fma(-u0, pp1, S.B01), X2 = fma(-u0, pp2, S.B02);
        const double zz0 = fma(x2, Z[2][0], fma(x1, Z[1][0], Z[0][0]));
        const double zz1 = fma(x2, Z[2][1], fma(x1, Z[1][1], Z[0][1]));
        const double zz2 = fma(x2, Z[2][2], fma(x1, Z[1][2], Z[0][2]));
        const double vb = dB == 0 ? v0 : (dB == 1 ? v1 : v2);
        const double zr0 = fma(-vb, zz0, dB == 0 ? Z[0][0] : (dB == 1 ? Z[1][0] : Z[2][0]));
        const double zr1 = fma(-vb, zz1, dB == 0 ? Z[0][1] : (dB == 1 ? Z[1][1] : Z[2][1]));
        const double zr2 = fma(-vb, zz2, dB == 0 ? Z[0][2] : (dB == 1 ? Z[1][2] : Z[2][2]));
        const bool own = ir >= k;
        const double c0 = spec ? zr0 : (own ? (d == 0 ? X0 : (d == 1 ? R10 : (d == 2 ? R20 : 0.0))) : b0);
        const double c1 = spec ? zr1 : (own ? (d == 0 ? X1 : (d == 1 ? R11 : (d == 2 ? R21 : 0.0))) : b1);
        const double c2 = spec ? zr2 : (own ? (d == 0 ? X2 : (d == 1 ? R12 : (d == 2 ? R22 : S.h3))) : b2);
        const double tt = fma(u2, c2, fma(u1, c1, u0 * c0));
        double* sc = dmy + HQ_SS * lane;
        *(cok ? rowp : sc) = c0 - tt;
        *(cok && k + 1 <= nn ? rowp + HQ_LD : sc + 1) = fma(-tt, w1, c1);
        *(cok && k + 2 <= nn ? rowp + 2 * HQ_LD : sc + 2) = fma(-tt, w2, c2);
      }
      {
        const double tq = fma(u2, g2, fma(u1, g1, u0 * g0));
        qp[0] = g0 - tq;
        qp[HQ_LD] = fma(-tq, w1, g1);
        qp[2 * HQ_LD] = fma(-tq, w2, g2);
      }
      S.B00 = N11; S.B01 = N12; S.B02 = R1c;
      S.B10 = N21; S.B11 = N22; S.B12 = R2c;
      S.B20 = N31; S.B21 = N32; S.B22 = S.d33;
      S.C0 = R1e; S.C1 = R2e; S.C2 = E3;
      S.h3 = h4; S.d33 = d44;
    }
    if (en && w > 0 && k + 1 == m) {  // this bulge enters next round, from the current matrix
      // (rows/cols m..m+2 are final: the bulge ahead is at m+3 and only touches indices >= m+3)
      const double z = H_(m, m), rr = sx - z, ss = sy - z;
      const double p = (rr * ss - sw) / H_(m + 1, m) + H_(m, m + 1);
      const double q = H_(m + 1, m + 1) - z - rr - ss;
      const double r = H_(m + 2, m + 1);
      load_state(m, S);
      S.B20 = 0.0;  // H[m+2][m]: zeroed by the bulge ahead (shared memory holds its stale entry)
      Rn = hq_refl_fast(p, q, r);
    }
    R = Rn;
    if (w > 0) put(R, (kA + 1) & 1);
    hq_barw(NWc);
  }
}

__device__ __forceinline__ void hq_chase2(double* Hw, double* Qs, double* dmy, int lo, int r1, int a0, int a1, int m,
                                          int nn, int l, double sp, double sq, double sr, double sx, double sy,
                                          double sw, int lane) {
  auto H_ = [&](int gi, int gj) -> double {
    return (gi >= lo && gj >= lo - 1 && gi <= r1 && gj <= r1) ? Hw[(gi - lo) + (gj - lo + 1) * HQ_LD] : 0.0;
  };
  auto load_state = [&](int k, HqBulge& S) {
    S.B00 = H_(k, k); S.B01 = H_(k, k + 1); S.B02 = H_(k, k + 2);
    S.B10 = H_(k + 1, k); S.B11 = H_(k + 1, k + 1); S.B12 = H_(k + 1, k + 2);
    S.B20 = H_(k + 2, k); S.B21 = H_(k + 2, k + 1); S.B22 = H_(k + 2, k + 2);
    S.C0 = H_(k, k + 3); S.C1 = H_(k + 1, k + 3); S.C2 = H_(k + 2, k + 3);
    S.h3 = H_(k + 3, k + 2); S.d33 = H_(k + 3, k + 3);
  };
  // first reflector input of a bulge at row k: the shift polynomial at m (NR's p, q, r; scale-free)
  // or the bulge column k-1
  auto intro = [&](int k, double& p, double& q, double& r) {
    const double z = H_(m, m), rr = sx - z, ss = sy - z;
    p = (rr * ss - sw) / H_(m + 1, m) + H_(m, m + 1);
    q = H_(m + 1, m + 1) - z - rr - ss;
    r = H_(m + 2, m + 1);
    (void)k;
  };
  // the second bulge only on active blocks long enough to hold both (short ones: one bulge)
  const bool twoB = nn - m >= HQ_TWO_MIN;
  HqBulge A = {}, Bb = {};
  HqRefl RA, RB;
  {
    const int kA = a0, kB = a0 - 4;
    double p, q, r;
    if (kA == m) {
      p = sp; q = sq; r = sr;
    } else {
      p = H_(kA, kA - 1); q = H_(kA + 1, kA - 1); r = H_(kA + 2, kA - 1);
    }
    if (kA <= nn - 1) {
      load_state(kA, A);
      RA = hq_refl_fast(p, q, r);
    } else {
      RA = hq_refl_fast(0.0, 0.0, 0.0);
    }
    if (twoB && kB >= m && kB <= nn - 1) {  // B already running: its bulge sits in column kB-1
      load_state(kB, Bb);
      RB = hq_refl_fast(H_(kB, kB - 1), H_(kB + 1, kB - 1), H_(kB + 2, kB - 1));
    } else {
      RB = hq_refl_fast(0.0, 0.0, 0.0);
    }
  }
  for (int kA = a0; kA < a1; ++kA) {
    const int kB = kA - 4;
    const bool actA = kA <= nn - 1, actB = twoB && kB >= m && kB <= nn - 1;
    if (kB == m && twoB) {  // introduce B from the current matrix (A has moved 4 positions)
      double p, q, r;
      intro(kB, p, q, r);
      load_state(kB, Bb);
      Bb.B20 = 0.0;  // H[m+2][m]: zeroed by A's step m+1 (shared memory still holds A's stale bulge entry)
      RB = hq_refl_fast(p, q, r);
    }
    // ---- loads (values after the previous round)
    const double E0 = H_(kA, kA + 4), E1 = H_(kA + 1, kA + 4), E2 = H_(kA + 2, kA + 4), E3 = H_(kA + 3, kA + 4);
    const double h4 = H_(kA + 4, kA + 3), d44 = H_(kA + 4, kA + 4);
    if (actB) {  // B's column k+3 and row k+3 are changed by A every round: reload
      Bb.C0 = H_(kB, kB + 3); Bb.C1 = H_(kB + 1, kB + 3); Bb.C2 = H_(kB + 2, kB + 3);
      Bb.h3 = H_(kB + 3, kB + 2); Bb.d33 = H_(kB + 3, kB + 3);
    }
    double Z[3][3];  // H[kB..kB+2][kA..kA+2]
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) Z[i][j] = H_(kB + i, kA + j);
    const int ir = lo + lane;  // this lane's row (column transforms, Q)
    // A row transformation: column kA+3+lane
    const int jA = kA + 3 + lane;
    const bool rokA = actA && jA <= r1;
    double* colA = rokA ? Hw + (jA - lo + 1) * HQ_LD + (kA - lo) : dmy + HQ_SS * lane;
    const double aA0 = colA[0], aA1 = colA[1], aA2 = colA[2];
    // B row transformation: column kB+3+lane, except A's columns kA..kA+2 (lanes 1..3)
    const int jB = kB + 3 + lane;
    const bool rokB = actB && jB <= r1 && (!actA || lane < 1 || lane > 3);
    double* colB = rokB ? Hw + (jB - lo + 1) * HQ_LD + (kB - lo) : dmy + HQ_SS * lane + 3;
    const double aB0 = colB[0], aB1 = colB[1], aB2 = colB[2];
    // A column transformation of row ir: loaded rows are those above kA outside B's rows
    const bool cokA = actA && ir <= min(nn, kA + 3);
    const bool specA = ir >= kB && ir <= kB + 2;
    const bool ldA = cokA && ir < kA && !specA;
    double* rowA = Hw + lane + (kA - lo + 1) * HQ_LD;
    const double bA0 = ldA ? rowA[0] : 0.0, bA1 = ldA ? rowA[HQ_LD] : 0.0, bA2 = ldA ? rowA[2 * HQ_LD] : 0.0;
    const bool cokB = actB && ir <= min(nn, kB + 3);
    const bool ldB = cokB && ir < kB;
    double* rowB = Hw + lane + (kB - lo + 1) * HQ_LD;
    const double bB0 = ldB ? rowB[0] : 0.0, bB1 = ldB ? rowB[HQ_LD] : 0.0, bB2 = ldB ? rowB[2 * HQ_LD] : 0.0;
    double* qA = Qs + lane + (actA ? kA - lo : 0) * HQ_LD;
    double* qB = Qs + lane + (actB ? kB - lo : 0) * HQ_LD;
    const double gA0 = qA[0], gA1 = qA[HQ_LD], gA2 = qA[2 * HQ_LD];
    const double gB0 = qB[0], gB1 = qB[HQ_LD], gB2 = qB[2 * HQ_LD];
    double* hkA = (lane == 0 && actA && RA.valid) ? Hw + (kA - lo) + (kA - lo) * HQ_LD : dmy + HQ_SS * lane + 6;
    double* hkB = (lane == 0 && actB && RB.valid) ? Hw + (kB - lo) + (kB - lo) * HQ_LD : dmy + HQ_SS * lane + 7;
    const double hkAv = *hkA, hkBv = *hkB;
    // ---- forward of A (as in the one-bulge chase)
    const double u0 = RA.xx, u1 = RA.yy, u2 = RA.zz, w1 = RA.qq, w2 = RA.rr;
    const double pp0 = fma(w2, A.B20, fma(w1, A.B10, A.B00)), pp1 = fma(w2, A.B21, fma(w1, A.B11, A.B01)),
                 pp2 = fma(w2, A.B22, fma(w1, A.B12, A.B02)), ppc = fma(w2, A.C2, fma(w1, A.C1, A.C0)),
                 ppe = fma(w2, E2, fma(w1, E1, E0));
    const double R10 = fma(-u1, pp0, A.B10), R11 = fma(-u1, pp1, A.B11), R12 = fma(-u1, pp2, A.B12),
                 R1c = fma(-u1, ppc, A.C1), R1e = fma(-u1, ppe, E1);
    const double R20 = fma(-u2, pp0, A.B20), R21 = fma(-u2, pp1, A.B21), R22 = fma(-u2, pp2, A.B22),
                 R2c = fma(-u2, ppc, A.C2), R2e = fma(-u2, ppe, E2);
    const double t1 = fma(u2, R12, fma(u1, R11, u0 * R10));
    const double t2 = fma(u2, R22, fma(u1, R21, u0 * R20));
    const double t3 = u2 * A.h3;
    const double N10 = R10 - t1, N11 = fma(-t1, w1, R11), N12 = fma(-t1, w2, R12);
    const double N20 = R20 - t2, N21 = fma(-t2, w1, R21), N22 = fma(-t2, w2, R22);
    const double N30 = -t3, N31 = -t3 * w1, N32 = fma(-t3, w2, A.h3);
    const HqRefl RnA = hq_refl_fast(actA && kA + 1 <= nn - 1 ? N10 : 0.0, actA && kA + 1 <= nn - 1 ? N20 : 0.0,
                                    actA && kA + 1 <= nn - 1 ? N30 : 0.0);
    // ---- forward of B
    const double v0 = RB.xx, v1 = RB.yy, v2 = RB.zz, x1 = RB.qq, x2 = RB.rr;
    const double qq0 = fma(x2, Bb.B20, fma(x1, Bb.B10, Bb.B00)), qq1 = fma(x2, Bb.B21, fma(x1, Bb.B11, Bb.B01)),
                 qq2 = fma(x2, Bb.B22, fma(x1, Bb.B12, Bb.B02)), qqc = fma(x2, Bb.C2, fma(x1, Bb.C1, Bb.C0));
    const double S10 = fma(-v1, qq0, Bb.B10), S11 = fma(-v1, qq1, Bb.B11), S12 = fma(-v1, qq2, Bb.B12),
                 S1c = fma(-v1, qqc, Bb.C1);
    const double S20 = fma(-v2, qq0, Bb.B20), S21 = fma(-v2, qq1, Bb.B21), S22 = fma(-v2, qq2, Bb.B22),
                 S2c = fma(-v2, qqc, Bb.C2);
    const double e1 = fma(v2, S12, fma(v1, S11, v0 * S10));
    const double e2 = fma(v2, S22, fma(v1, S21, v0 * S20));
    const double e3 = v2 * Bb.h3;
    const double M10 = S10 - e1, M11 = fma(-e1, x1, S11), M12 = fma(-e1, x2, S12);
    const double M20 = S20 - e2, M21 = fma(-e2, x1, S21), M22 = fma(-e2, x2, S22);
    const double M30 = -e3, M31 = -e3 * x1, M32 = fma(-e3, x2, Bb.h3);
    const bool nxB = actB && kB + 1 <= nn - 1;
    const HqRefl RnB = hq_refl_fast(nxB ? M10 : 0.0, nxB ? M20 : 0.0, nxB ? M30 : 0.0);
    // ---- shared-memory updates of the round (masked lanes write to their scratch slots)
    *hkA = (kA == m) ? ((l != m) ? -hkAv : hkAv) : -RA.s;
    *hkB = (kB == m) ? ((l != m) ? -hkBv : hkBv) : -RB.s;
    {  // row transformations
      const double prA = fma(w2, aA2, fma(w1, aA1, aA0));
      colA[0] = fma(-u0, prA, aA0);
      colA[1] = fma(-u1, prA, aA1);
      *((rokA && kA + 2 <= nn) ? colA + 2 : dmy + HQ_SS * lane + 2) = fma(-u2, prA, aA2);
      const double prB = fma(x2, aB2, fma(x1, aB1, aB0));
      colB[0] = fma(-v0, prB, aB0);
      colB[1] = fma(-v1, prB, aB1);
      *((rokB && kB + 2 <= nn) ? colB + 2 : dmy + HQ_SS * lane + 5) = fma(-v2, prB, aB2);
    }
    {  // A's column transformation (cols kA..kA+2)
      const int d = ir - kA, dB = ir - kB;
      const double X0 = fma(-u0, pp0, A.B00), X1 = fma(-u0, pp1, A.B01), X2 = fma(-u0, pp2, A.B02);
      // B's rows: P_B from the left on the Z block first
      const double zz0 = fma(x2, Z[2][0], fma(x1, Z[1][0], Z[0][0]));
      const double zz1 = fma(x2, Z[2][1], fma(x1, Z[1][1], Z[0][1]));
      const double zz2 = fma(x2, Z[2][2], fma(x1, Z[1][2], Z[0][2]));
      const double vb = dB == 0 ? v0 : (dB == 1 ? v1 : v2);
      const double zr0 = fma(-vb, zz0, dB == 0 ? Z[0][0] : (dB == 1 ? Z[1][0] : Z[2][0]));
      const double zr1 = fma(-vb, zz1, dB == 0 ? Z[0][1] : (dB == 1 ? Z[1][1] : Z[2][1]));
      const double zr2 = fma(-vb, zz2, dB == 0 ? Z[0][2] : (dB == 1 ? Z[1][2] : Z[2][2]));
      const bool own = ir >= kA;
      const double c0 = specA ? zr0 : (own ? (d == 0 ? X0 : (d == 1 ? R10 : (d == 2 ? R20 : 0.0))) : bA0);
      const double c1 = specA ? zr1 : (own ? (d == 0 ? X1 : (d == 1 ? R11 : (d == 2 ? R21 : 0.0))) : bA1);
      const double c2 = specA ? zr2 : (own ? (d == 0 ? X2 : (d == 1 ? R12 : (d == 2 ? R22 : A.h3))) : bA2);
      const double tt = fma(u2, c2, fma(u1, c1, u0 * c0));
      // the special block exists only where both columns and rows are real (<= nn, in the window)
      const bool stA = cokA;
      double* sc = dmy + HQ_SS * lane;
      *(stA ? rowA : sc) = c0 - tt;
      *(stA && kA + 1 <= nn ? rowA + HQ_LD : sc + 1) = fma(-tt, w1, c1);
      *(stA && kA + 2 <= nn ? rowA + 2 * HQ_LD : sc + 2) = fma(-tt, w2, c2);
    }
    {  // B's column transformation (cols kB..kB+2)
      const int d = ir - kB;
      const double Y0 = fma(-v0, qq0, Bb.B00), Y1 = fma(-v0, qq1, Bb.B01), Y2 = fma(-v0, qq2, Bb.B02);
      const bool own = ir >= kB;
      const double c0 = own ? (d == 0 ? Y0 : (d == 1 ? S10 : (d == 2 ? S20 : 0.0))) : bB0;
      const double c1 = own ? (d == 0 ? Y1 : (d == 1 ? S11 : (d == 2 ? S21 : 0.0))) : bB1;
      const double c2 = own ? (d == 0 ? Y2 : (d == 1 ? S12 : (d == 2 ? S22 : Bb.h3))) : bB2;
      const double tt = fma(v2, c2, fma(v1, c1, v0 * c0));
      double* sc = dmy + HQ_SS * lane + 3;
      *(cokB ? rowB : sc) = c0 - tt;
      *(cokB ? rowB + HQ_LD : sc + 1) = fma(-tt, x1, c1);
      *((cokB && kB + 2 <= nn) ? rowB + 2 * HQ_LD : sc + 2) = fma(-tt, x2, c2);
    }
    {  // Q <- Q P_A P_B (disjoint columns; an inactive bulge's stores go to scratch, not over the other's)
      double* sq = dmy + HQ_SS * lane + 8;
      const double tqA = fma(u2, gA2, fma(u1, gA1, u0 * gA0));
      *(actA ? qA : sq) = gA0 - tqA;
      *(actA ? qA + HQ_LD : sq + 1) = fma(-tqA, w1, gA1);
      *(actA ? qA + 2 * HQ_LD : sq + 2) = fma(-tqA, w2, gA2);
      const double tqB = fma(v2, gB2, fma(v1, gB1, v0 * gB0));
      *(actB ? qB : sq + 3) = gB0 - tqB;
      *(actB ? qB + HQ_LD : sq + 4) = fma(-tqB, x1, gB1);
      *(actB ? qB + 2 * HQ_LD : sq + 5) = fma(-tqB, x2, gB2);
    }
    __syncwarp();
    RA = RnA;
    A.B00 = N11; A.B01 = N12; A.B02 = R1c;
    A.B10 = N21; A.B11 = N22; A.B12 = R2c;
    A.B20 = N31; A.B21 = N32; A.B22 = A.d33;
    A.C0 = R1e; A.C1 = R2e; A.C2 = E3;
    A.h3 = h4; A.d33 = d44;
    RB = RnB;
    Bb.B00 = M11; Bb.B01 = M12; Bb.B02 = S1c;
    Bb.B10 = M21; Bb.B11 = M22; Bb.B12 = S2c;
    Bb.B20 = M31; Bb.B21 = M32; Bb.B22 = Bb.d33;
  }
}

__global__ void __launch_bounds__(HQ_THREADS) hqr_kernel(double* __restrict__ a, int n, int lda,
                                                         double* __restrict__ wr, double* __restrict__ wi,
                                                         int* __restrict__ info) {
  __shared__ double Hw[HQ_LD * (HQ_R + 1) + HQ_SS * 32];  // window + per-lane scratch
#if HQ_XPF && HQ_NB == 3
  __shared__ double Hw2[HQ_LD * (HQ_R + 1)];  // the other window buffer
  __shared__ double Xb[HQ_R * (HQ_R - 3)];    // prefetched H[window rows][next window's new columns]
#endif
  __shared__ double Qsh[2 * HQ_QSZ];  // accumulated Q of the current / previous window
  __shared__ double hq_x[16 * 8];     // HQ_NB=3: each chase warp's next reflector, by round parity
  __shared__ double red[32];
  __shared__ int ired[32];
  __shared__ double sp, sq, sr, sx, sy, sw, st;
  __shared__ int sl, snn, sm, sflag, sits, sdone, nsweep, nstep;
  long long cyc_chase = 0, cyc_all = clock64();
#ifdef HQ_PROF
  long long cyc_setup = 0, cyc_trans = 0, cyc_last = 0;
#endif
  const int tid = threadIdx.x, nt = blockDim.x;
  // anorm
  double loc = 0.0;
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += nt) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    if (j >= i - 1) loc += fabs(HA(i, j));
  }
  const double anorm0 = block_sum(loc, red);
  // scale by a power of two so that ||H||_1-ish ~ 1 (exact; the eigenvalues are scaled back at the
  // end): the reflectors of the sweep then never leave the normal exponent range
  const double hsc = anorm0 > 0.0 ? ldexp(1.0, -ilogb(anorm0)) : 1.0;
  const double anorm = anorm0 * hsc;
  for (int64_t idx = tid; idx < (int64_t)n * n; idx += nt) {
    const int i = (int)(idx % n), j = (int)(idx / n);
    HA(i, j) *= hsc;
  }
  __syncthreads();
  if (tid == 0) {
    snn = n - 1;
    st = 0.0;
    sdone = 0;
    nsweep = 0;
    nstep = 0;
  }
  __syncthreads();
  while (true) {
    if (snn < 0) break;
    if (tid == 0) sits = 0;
    __syncthreads();
    while (true) {
#ifdef HQ_PROF
      const long long tp0 = clock64();
#endif
#ifdef HQ_DEBUG_SWEEPS  // debugging harness: stop after info[7] sweeps (if > 0), H left in place
      if (info[7] > 0 && nsweep >= info[7]) {
        __syncthreads();
        if (tid == 0) sdone = 1;
        __syncthreads();
        break;
      }
#endif
      // --- find the largest l in [1, nn] with a negligible subdiagonal (all threads, one pass
      //     over the subdiagonal instead of a serial scan with one L2 round trip per element)
      {
        const int nn = snn;
        int best = 0;
        for (int l = 1 + tid; l <= nn; l += nt) {
          double s = fabs(HA(l - 1, l - 1)) + fabs(HA(l, l));
          if (s == 0.0) s = anorm;
          if (fabs(HA(l, l - 1)) + s == s) best = max(best, l);
        }
        best = block_max_int(best, ired);
        if (tid == 0) sl = best;
      }
      __syncthreads();
      // --- scalar part: deflate or set up a double-shift sweep
      if (tid == 0) {
        int nn = snn, l = sl;
        if (l >= 1) HA(l, l - 1) = 0.0;
        double x = HA(nn, nn);
        sflag = 0;
        if (l == nn) {
          wr[nn] = x + st;
          wi[nn] = 0.0;
          snn = nn - 1;
        } else {
          double y = HA(nn - 1, nn - 1);
          double w = HA(nn, nn - 1) * HA(nn - 1, nn);
          if (l == nn - 1) {
            double p = 0.5 * (y - x);
            double q = p * p + w;
            double z = sqrt(fabs(q));
            x += st;
            if (q >= 0.0) {
              z = p + copysign(z, p);
              wr[nn - 1] = wr[nn] = x + z;
              if (z != 0.0) wr[nn] = x - w / z;
              wi[nn - 1] = wi[nn] = 0.0;
            } else {
              wr[nn - 1] = wr[nn] = x + p;
              wi[nn] = z;
              wi[nn - 1] = -z;
            }
            snn = nn - 2;
          } else {
            if (sits >= 60) {
              info[0] = 1;  // no convergence
              sdone = 1;
            } else {
              if (sits > 0 && sits % 10 == 0) {  // exceptional shift
                sflag = 2;
                sx = x;
              } else {
                sflag = 1;
              }
              sx = x;
              sy = y;
              sw = w;
            }
          }
        }
        sl = l;
      }
      __syncthreads();
      if (sdone) break;
      if (sflag == 0) {  // deflated
        const int nn = snn, l = sl;
        __syncthreads();
        if (!(l < nn - 1)) break;  // leave inner loop (reset iteration count)
        continue;
      }
      if (sflag == 2) {
        const double x = sx;
        for (int i = tid; i <= snn; i += nt) HA(i, i) -= x;
        __syncthreads();
        if (tid == 0) {
          const int nn = snn;
          st += x;
          double s = fabs(HA(nn, nn - 1)) + fabs(HA(nn - 1, nn - 2));
          sx = sy = 0.75 * s;
          sw = -0.4375 * s * s;
        }
        __syncthreads();
      }
      // choose m (largest m in [l, nn-2] with m == l or two small consecutive subdiagonals,
      // evaluated for all m in parallel) and the first Householder vector
      {
        const int nn = snn, l = sl;
        const double x = sx, y = sy, w = sw;
        auto pqr = [&](int m, double& p, double& q, double& r, double& z) {
          z = HA(m, m);
          r = x - z;
          double s = y - z;
          p = (r * s - w) / HA(m + 1, m) + HA(m, m + 1);
          q = HA(m + 1, m + 1) - z - r - s;
          r = HA(m + 2, m + 1);
          s = fabs(p) + fabs(q) + fabs(r);
          p /= s;
          q /= s;
          r /= s;
        };
        int best = l;
        for (int m = l + 1 + tid; m <= nn - 2; m += nt) {
          double p, q, r, z;
          pqr(m, p, q, r, z);
          const double u = fabs(HA(m, m - 1)) * (fabs(q) + fabs(r));
          const double v = fabs(p) * (fabs(HA(m - 1, m - 1)) + fabs(z) + fabs(HA(m + 1, m + 1)));
          if (u + v == v) best = max(best, m);
        }
        best = block_max_int(best, ired);
        if (tid == 0) {
          sits = sits + 1;
          double p, q, r, z;
          pqr(best, p, q, r, z);
          sm = best;
          nsweep += 1;
          nstep += nn - best;
          sp = p;
          sq = q;
          sr = r;
        }
      }
      __syncthreads();
      {
        const int nn = snn, m = sm;
        for (int i = m + 2 + tid; i <= nn; i += nt) {
          HA(i, i - 2) = 0.0;
          if (i != m + 2) HA(i, i - 3) = 0.0;
        }
      }
      __syncthreads();
      // --- the double-shift sweep k = m .. nn-1, chased through windows of HQ_W steps.
      //     Window rows/cols R = [k0, r1] (r1 <= k0+31) live in shared memory (Hw, column k0-1
      //     included for the reflector reads); warp 0 chases the bulge through them with warp-level
      //     syncs only, applying each 3x3 reflector P_k exactly as the per-element sweep does inside
      //     the window and accumulating Q = P_k0 ... P_k1-1.  The parts of P_k's row/column
      //     transformations outside the window are applied afterwards as one block update by the
      //     whole CTA: H[R, (r1, nn]] <- Q^T H[R, (r1, nn]],  H[[l, k0), R] <- H[[l, k0), R] Q.
      //     Same reflectors, same order; only the rounding of the far updates differs.
      const int nn = snn, l = sl, m = sm;
      const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
      // Off-window block update with the accumulated Q of a window [wk0, wr1] (FP64 tensor cores,
      // mma.m8n8k4.f64; a warp per 8-vector tile, the 32x32 Q held as 32 fragments per thread:
      // frag[t][ks] = Q[4ks + lane%4, 8t + lane/4], the A fragment of Q^T and the B fragment of Q):
      //   right part, columns (clo, chi]:  H[R, c]  <- Q^T H[R, c]
      //   above part, rows [alo, ahi):     H[i, R]  <- H[i, R] Q
      auto far_update = [&](const double* qb, int wk0, int wr1, int clo, int chi, int alo, int ahi, int w0,
                            int ws) {
        const int wnr = wr1 - wk0 + 1;
        const int lr = lane >> 2, lc = lane & 3;
        const int ncol = chi - clo, nrow = ahi - alo;
        const int ntc = ncol > 0 ? (ncol + 7) >> 3 : 0, ntr = nrow > 0 ? (nrow + 7) >> 3 : 0;
        // w0 < 0: deferred mode, workers are the warps off the chasing warps' schedulers
        int me = warp - w0;
        if (w0 < 0) {
#if HQ_NB == 3
          if (HQ_NW <= 2) {
            if ((warp & 3) < 2) return;  // warps 0, 1 chase; 4, 5, 8, 9 share their schedulers
            me = (warp >> 2) * 2 + (warp & 3) - 2;
          } else {  // every scheduler has a chase warp: all other warps work
            if (warp < HQ_NW) return;
            me = warp - HQ_NW;
          }
#else
          if ((warp & 3) == 0) return;
          me = warp - (warp >> 2) - 1;
#endif
        }
        if (me < 0 || me >= ntc + ntr) return;
        double fq[4][8];
#pragma unroll
        for (int t = 0; t < 4; ++t)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) fq[t][ks] = qb[4 * ks + lc + (8 * t + lr) * HQ_LD];
        for (int u = me; u < ntc + ntr; u += ws) {
          double fx[8], d[4][2];
#pragma unroll
          for (int t = 0; t < 4; ++t) d[t][0] = d[t][1] = 0.0;
          if (u < ntc) {
            const int c = 8 * u + lr;  // B fragment: H[wk0 + 4ks + lc, clo + 1 + c]
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int k = 4 * ks + lc;
              fx[ks] = (c < ncol && k < wnr) ? HA(wk0 + k, clo + 1 + c) : 0.0;
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
              for (int t = 0; t < 4; ++t) dmma884(d[t][0], d[t][1], fq[t][ks], fx[ks]);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const int mm = 8 * t + lr;
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int cc = 8 * u + 2 * lc + e;
                if (mm < wnr && cc < ncol) HA(wk0 + mm, clo + 1 + cc) = d[t][e];
              }
            }
          } else {
            const int i = alo + 8 * (u - ntc) + lr;  // A fragment: H[i, wk0 + 4ks + lc]
#pragma unroll
            for (int ks = 0; ks < 8; ++ks) {
              const int k = 4 * ks + lc;
              fx[ks] = (i < ahi && k < wnr) ? HA(i, wk0 + k) : 0.0;
            }
#pragma unroll
            for (int ks = 0; ks < 8; ++ks)
#pragma unroll
              for (int t = 0; t < 4; ++t) dmma884(d[t][0], d[t][1], fx[ks], fq[t][ks]);
#pragma unroll
            for (int t = 0; t < 4; ++t)
#pragma unroll
              for (int e = 0; e < 2; ++e) {
                const int nc = 8 * t + 2 * lc + e;
                if (i < ahi && nc < wnr) HA(i, wk0 + nc) = d[t][e];
              }
          }
        }
      };
      auto load_window = [&](int wk0, int wr1, double* qb) {
        const int wnr = wr1 - wk0 + 1;
        for (int idx = tid; idx < HQ_R * (HQ_R + 1); idx += nt) {
          const int i = idx % HQ_R, c = idx / HQ_R;  // local row i = wk0+i, local col c = wk0-1+c
          const int gj = wk0 - 1 + c;
          Hw[i + c * HQ_LD] = (i < wnr && gj >= 0 && gj <= wr1) ? HA(wk0 + i, gj) : 0.0;
        }
        for (int idx = tid; idx < HQ_R * HQ_R; idx += nt) {
          const int i = idx % HQ_R, c = idx / HQ_R;
          qb[i + c * HQ_LD] = (i == c) ? 1.0 : 0.0;
        }
      };
      // Pipeline over the windows of the sweep: while warp 0 chases window w, the other warps apply
      // the deferred off-window update of window w-1 (its columns beyond window w and its rows
      // above); the part of w's update that window w+1 reads (its columns) is done before w+1 loads.
      int k0 = m;  // window rows/cols [k0, r1]
#if HQ_NB == 3
      const int hspan = 4 * (hq_nbulges(nn, m) - 1);  // rows between the first and the last bulge
#else
      const int hspan = 4;
#endif
#if HQ_NB >= 2
      int a0 = m, a1 = min(k0 + HQ_R - 3, nn + hspan);  // rounds: bulge 0 at kA in [a0, a1), bulge w at kA - 4w
      int k1 = a1;
#else
      int k1 = min(k0 + HQ_W, nn);
#endif
      int r1 = min(k0 + HQ_R - 1, nn);
      int cur = 0, pk0 = -1, pr1 = 0;
      double* Hc = Hw;  // the current window's buffer
#if HQ_XPF && HQ_NB == 3
      const bool sp_ok = (HQ_NW <= 2) ? ((warp & 3) >= 2) : (warp >= HQ_NW);  // warps off the chase schedulers
      const int sp_t = (HQ_NW <= 2) ? (((warp >> 2) * 2 + (warp & 3) - 2) * 32 + lane) : ((warp - HQ_NW) * 32 + lane);
      const int sp_n = (HQ_NW <= 2) ? (nw / 2) * 32 : (nw - HQ_NW) * 32;
#endif
      load_window(k0, r1, Qsh);
      __syncthreads();
#ifdef HQ_PROF
      if (tid == 0) cyc_setup += clock64() - tp0;
#endif
      while (true) {
        double* Qs = Qsh + cur * HQ_QSZ;
        long long tc0 = clock64();
#if HQ_NB == 3
        if (warp < HQ_NW) {
          // two bulges: the role-specialised chase; more: the general one (correct, but every warp then
          // issues the union of both roles' work: C5 hqr 33 ms at 4 bulges vs 27.6 ms here)
          if (HQ_NW == 2)
            hq_chase2w(Hc, Qs, Hw + HQ_LD * (HQ_R + 1), hq_x, k0, r1, a0, a1, m, nn, l, sp, sq, sr, sx, sy, sw, lane,
                       warp);
          else
            hq_chasew(Hc, Qs, Hw + HQ_LD * (HQ_R + 1), hq_x, k0, r1, a0, a1, m, nn, l, sp, sq, sr, sx, sy, sw, lane,
                      warp);
        }
#if HQ_XPF
        else if (sp_ok) {  // spare warps: pending write-back, deferred off-window update, next-window prefetch
          double* Hn = (Hc == Hw) ? Hw2 : Hw;  // the previous window's buffer = the next window's
          if (pk0 >= 0) {
            for (int idx = sp_t; idx < HQ_R * (HQ_R + 1); idx += sp_n) {  // write the previous window back
              const int i = idx % HQ_R, c = idx / HQ_R;
              const int gj = pk0 - 1 + c;
              if (i <= pr1 - pk0 && gj >= 0 && gj <= pr1) HA(pk0 + i, gj) = Hn[i + c * HQ_LD];
            }
            far_update(Qsh + (cur ^ 1) * HQ_QSZ, pk0, pr1, r1, nn, l, pk0, -1, HQ_NW <= 2 ? nw / 2 : nw - HQ_NW);
            __threadfence_block();
            asm volatile("bar.sync 2, %0;" ::"r"(sp_n) : "memory");
          }
          const int k0n = a1 - hspan;
          if (a1 < nn + hspan) {  // not the last window: prefetch for window [k0n, r1n]
            const int r1n = min(k0n + HQ_R - 1, nn), ncx = r1n - r1, wnr = r1 - k0 + 1;
            for (int idx = sp_t; idx < wnr * ncx; idx += sp_n) {
              const int i = idx % wnr, c = idx / wnr;
              Xb[i + c * HQ_R] = HA(k0 + i, r1 + 1 + c);
            }
            // rows below this window (local rows > r1 - k0n of the next window), every local column; zeros
            // beyond the active block; also zero the next window's columns beyond r1n on the overlap rows
            for (int idx = sp_t; idx < HQ_R * (HQ_R + 1); idx += sp_n) {
              const int i = idx % HQ_R, c = idx / HQ_R;
              const int gi = k0n + i, gj = k0n - 1 + c;
              if (gi > r1) Hn[i + c * HQ_LD] = (gi <= r1n && gj >= 0 && gj <= r1n) ? HA(gi, gj) : 0.0;
              else if (gj > r1n) Hn[i + c * HQ_LD] = 0.0;
            }
          }
        }
#endif
#elif HQ_NB == 2
        if (warp == 0) {
          hq_chase2(Hw, Qs, Hw + HQ_LD * (HQ_R + 1), k0, r1, a0, a1, m, nn, l, sp, sq, sr, sx, sy, sw, lane);
        }
#else
        if (warp == 0) {
          // Register-forwarded chase.  Every lane carries the step's reflector and the bulge state
          // (B = H[k..k+2][k..k+2], C = H[k..k+2][k+3], h3 = H[k+3][k+2], d33 = H[k+3][k+3]) and
          // derives step k+1's reflector input H[k+1..k+3][k] (and state) from them in registers,
          // so the dependent chain per step is reflector -> 3x3 update -> reflector; the shared
          // memory updates of step k (one phase: the 3x3 block rows come from the registers) and
          // the Q update run alongside.  Entries beyond the window / active block read as 0.
          auto H_ = [&](int gi, int gj) -> double {
            return (gi <= r1 && gj <= r1) ? Hw[(gi - k0) + (gj - k0 + 1) * HQ_LD] : 0.0;
          };
          int k = k0;
          double p0_, q0_, r0_;
          if (k == m) {
            p0_ = sp;
            q0_ = sq;
            r0_ = sr;
          } else {
            p0_ = H_(k, k - 1);
            q0_ = H_(k + 1, k - 1);
            r0_ = H_(k + 2, k - 1);
          }
          double B00 = H_(k, k), B01 = H_(k, k + 1), B02 = H_(k, k + 2);
          double B10 = H_(k + 1, k), B11 = H_(k + 1, k + 1), B12 = H_(k + 1, k + 2);
          double B20 = H_(k + 2, k), B21 = H_(k + 2, k + 1), B22 = H_(k + 2, k + 2);
          double C0 = H_(k, k + 3), C1 = H_(k + 1, k + 3), C2 = H_(k + 2, k + 3);
          double h3 = H_(k + 3, k + 2), d33 = H_(k + 3, k + 3);
          HqRefl R = hq_refl_fast(p0_, q0_, r0_);
          double* dmy = Hw + HQ_LD * (HQ_R + 1);  // scratch for masked stores (4 doubles per lane)
          for (; k < k1; ++k) {
            const int kk = k - k0;
            // ---- loads (values after step k-1).  One basic block per step: the shared-memory
            //      updates of step k interleave with the register chain of step k+1.  Loaded
            //      values are stored back (updated) only by the lane that loaded them, except
            //      E0..E2, read by all lanes before lane 1 (column k+4) stores them (same
            //      warp-converged instruction stream).
            const double E0 = H_(k, k + 4), E1 = H_(k + 1, k + 4), E2 = H_(k + 2, k + 4), E3 = H_(k + 3, k + 4);
            const double h4 = H_(k + 4, k + 3), d44 = H_(k + 4, k + 4);
            const int jr = k + 3 + lane;  // row transformation: this lane's column
            const bool rok = jr <= r1;
            double* colr = rok ? Hw + (jr - k0 + 1) * HQ_LD + kk : dmy + 4 * lane;
            const double a0 = colr[0], a1 = colr[1], a2 = colr[2];
            const int ir = k0 + lane;  // column transformation: this lane's row
            const bool cok = ir <= min(nn, k + 3), above = ir < k;
            double* rowc = (cok && above) ? Hw + lane + (kk + 1) * HQ_LD : dmy + 4 * lane;
            const double b0 = rowc[0], b1 = rowc[above && cok ? HQ_LD : 1], b2 = rowc[above && cok ? 2 * HQ_LD : 2];
            double* qc = Qs + lane + kk * HQ_LD;
            const double g0 = qc[0], g1 = qc[HQ_LD], g2 = qc[2 * HQ_LD];
            double* hk = (lane == 0 && R.valid) ? Hw + kk + kk * HQ_LD : dmy + 4 * lane + 3;  // H(k, k-1)
            const double hkv = *hk;
            const double u0 = R.xx, u1 = R.yy, u2 = R.zz, w1 = R.qq, w2 = R.rr;
            // ---- forward: H' = (I - u w^T) H on rows k..k+2, then the column update of rows k+1..k+3
            const double pp0 = fma(w2, B20, fma(w1, B10, B00)), pp1 = fma(w2, B21, fma(w1, B11, B01)),
                         pp2 = fma(w2, B22, fma(w1, B12, B02)), ppc = fma(w2, C2, fma(w1, C1, C0)),
                         ppe = fma(w2, E2, fma(w1, E1, E0));
            const double R10 = fma(-u1, pp0, B10), R11 = fma(-u1, pp1, B11), R12 = fma(-u1, pp2, B12),
                         R1c = fma(-u1, ppc, C1), R1e = fma(-u1, ppe, E1);
            const double R20 = fma(-u2, pp0, B20), R21 = fma(-u2, pp1, B21), R22 = fma(-u2, pp2, B22),
                         R2c = fma(-u2, ppc, C2), R2e = fma(-u2, ppe, E2);
            const double t1 = fma(u2, R12, fma(u1, R11, u0 * R10));
            const double t2 = fma(u2, R22, fma(u1, R21, u0 * R20));
            const double t3 = u2 * h3;
            const double N10 = R10 - t1, N11 = fma(-t1, w1, R11), N12 = fma(-t1, w2, R12);
            const double N20 = R20 - t2, N21 = fma(-t2, w1, R21), N22 = fma(-t2, w2, R22);
            const double N30 = -t3, N31 = -t3 * w1, N32 = fma(-t3, w2, h3);
            const HqRefl Rn = hq_refl_fast(N10, N20, N30);
            // ---- shared-memory updates of step k (masked lanes write to their scratch slots)
            *hk = (k == m) ? ((l != m) ? -hkv : hkv) : -R.s;
            {
              const double pr = fma(w2, a2, fma(w1, a1, a0));
              colr[0] = fma(-u0, pr, a0);
              colr[1] = fma(-u1, pr, a1);
              *((k + 2 <= nn) ? colr + 2 : dmy + 4 * lane + 2) = fma(-u2, pr, a2);
            }
            {
              const int d = ir - k;
              const double X0 = fma(-u0, pp0, B00), X1 = fma(-u0, pp1, B01), X2 = fma(-u0, pp2, B02);
              const double v0 = above ? b0 : (d == 0 ? X0 : (d == 1 ? R10 : (d == 2 ? R20 : 0.0)));
              const double v1 = above ? b1 : (d == 0 ? X1 : (d == 1 ? R11 : (d == 2 ? R21 : 0.0)));
              const double v2 = above ? b2 : (d == 0 ? X2 : (d == 1 ? R12 : (d == 2 ? R22 : h3)));
              const double tt = fma(u2, v2, fma(u1, v1, u0 * v0));
              double* rw = Hw + lane + (kk + 1) * HQ_LD;
              double* sc = dmy + 4 * lane;
              *(cok ? rw : sc) = v0 - tt;
              *(cok ? rw + HQ_LD : sc + 1) = fma(-tt, w1, v1);
              *((cok && k + 2 <= nn) ? rw + 2 * HQ_LD : sc + 2) = fma(-tt, w2, v2);
            }
            {
              const double tq = fma(u2, g2, fma(u1, g1, u0 * g0));
              qc[0] = g0 - tq;
              qc[HQ_LD] = fma(-tq, w1, g1);
              qc[2 * HQ_LD] = fma(-tq, w2, g2);
            }
            __syncwarp();
            R = Rn;
            B00 = N11;
            B01 = N12;
            B02 = R1c;
            B10 = N21;
            B11 = N22;
            B12 = R2c;
            B20 = N31;
            B21 = N32;
            B22 = d33;
            C0 = R1e;
            C1 = R2e;
            C2 = E3;
            h3 = h4;
            d33 = d44;
          }
        }
#endif
#if !(HQ_XPF && HQ_NB == 3)
        else if (pk0 >= 0) {
          far_update(Qsh + (cur ^ 1) * HQ_QSZ, pk0, pr1, r1, nn, l, pk0, -1,
                     HQ_NB == 3 ? (HQ_NW <= 2 ? nw / 2 : nw - HQ_NW) : nw - (nw >> 2));
        }
#endif
        __syncthreads();
        long long tc1 = clock64();
        if (tid == 0) cyc_chase += tc1 - tc0;
#if HQ_XPF && HQ_NB == 3
        {
          const int k0n = a1 - hspan;  // the next window starts at the last bulge's row
          if (a1 >= nn + hspan) {      // last window: write back, its whole off-window update now
            for (int idx = tid; idx < HQ_R * (HQ_R + 1); idx += nt) {
              const int i = idx % HQ_R, c = idx / HQ_R;
              const int gj = k0 - 1 + c;
              if (i <= r1 - k0 && gj >= 0 && gj <= r1) HA(k0 + i, gj) = Hc[i + c * HQ_LD];
            }
            far_update(Qs, k0, r1, r1, nn, l, k0, 0, nw);
            __syncthreads();
#ifdef HQ_PROF
            if (tid == 0) cyc_last += clock64() - tc1;
#endif
            break;
          }
          const int r1n = min(k0n + HQ_R - 1, nn), ncx = r1n - r1, wnr = r1 - k0 + 1;
          double* Hn = (Hc == Hw) ? Hw2 : Hw;
          // next window's new columns (r1, r1n] on this window's rows: Q^T Xb (global: rows above the next window)
          for (int idx = tid; idx < wnr * ncx; idx += nt) {
            const int i = idx % wnr, c = idx / wnr;
            const double* qi = Qs + i * HQ_LD;
            const double* xc = Xb + c * HQ_R;
            double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;
            int kq = 0;
            for (; kq + 3 < wnr; kq += 4) {
              z0 = fma(qi[kq], xc[kq], z0);
              z1 = fma(qi[kq + 1], xc[kq + 1], z1);
              z2 = fma(qi[kq + 2], xc[kq + 2], z2);
              z3 = fma(qi[kq + 3], xc[kq + 3], z3);
            }
            for (; kq < wnr; ++kq) z0 = fma(qi[kq], xc[kq], z0);
            const double z = (z0 + z1) + (z2 + z3);
            const int gi = k0 + i, gj = r1 + 1 + c;
            HA(gi, gj) = z;
            if (gi >= k0n) Hn[(gi - k0n) + (gj - k0n + 1) * HQ_LD] = z;
          }
          // the overlap block rows/cols [k0n, r1] (and column k0n - 1) from this window
          for (int idx = tid; idx < HQ_R * (HQ_R + 1); idx += nt) {
            const int i = idx % HQ_R, c = idx / HQ_R;
            const int gi = k0n + i, gj = k0n - 1 + c;
            if (gi <= r1 && gj <= r1) Hn[i + c * HQ_LD] = Hc[(gi - k0) + (gj - k0 + 1) * HQ_LD];
          }
          double* qn = Qsh + (cur ^ 1) * HQ_QSZ;  // the previous window's Q (its deferred update is done)
          for (int idx = tid; idx < HQ_R * HQ_R; idx += nt) {
            const int i = idx % HQ_R, c = idx / HQ_R;
            qn[i + c * HQ_LD] = (i == c) ? 1.0 : 0.0;
          }
          __syncthreads();
          pk0 = k0;
          pr1 = r1;
          cur ^= 1;
          k0 = k0n;
          a0 = a1;
          a1 = min(k0 + HQ_R - 3, nn + hspan);
          k1 = a1;
          r1 = r1n;
          Hc = Hn;
#ifdef HQ_PROF
          if (tid == 0) cyc_trans += clock64() - tc1;
#endif
          continue;
        }
#endif
        for (int idx = tid; idx < HQ_R * (HQ_R + 1); idx += nt) {  // write the window back
          const int i = idx % HQ_R, c = idx / HQ_R;
          const int gj = k0 - 1 + c;
          if (i <= r1 - k0 && gj >= 0 && gj <= r1) HA(k0 + i, gj) = Hw[i + c * HQ_LD];
        }
#if HQ_NB >= 2
        const int k0n = a1 - hspan;  // the next window starts at the last bulge's row
        if (a1 >= nn + hspan) {      // last window: its whole off-window update now
#else
        const int k0n = k1;
        if (k0n > nn - 1) {  // last window: its whole off-window update now
#endif
          far_update(Qs, k0, r1, r1, nn, l, k0, 0, nw);
          __syncthreads();
#ifdef HQ_PROF
          if (tid == 0) cyc_last += clock64() - tc1;
#endif
          break;
        }
        const int r1n = min(k0n + HQ_R - 1, nn);
        far_update(Qs, k0, r1, r1, r1n, 0, 0, 0, nw);  // the next window's columns
        __syncthreads();
        pk0 = k0;
        pr1 = r1;
        cur ^= 1;
        k0 = k0n;
#if HQ_NB >= 2
        a0 = a1;
        a1 = min(k0 + HQ_R - 3, nn + hspan);
        k1 = a1;
#else
        k1 = min(k0 + HQ_W, nn);
#endif
        r1 = r1n;
        load_window(k0, r1, Qsh + cur * HQ_QSZ);
        __syncthreads();
#ifdef HQ_PROF
        if (tid == 0) cyc_trans += clock64() - tc1;
#endif
      }
      {
        const int nn2 = snn, l2 = sl;
        __syncthreads();
        if (!(l2 < nn2 - 1)) break;
      }
    }
    if (sdone) break;
  }
  __syncthreads();
  const double ihsc = 1.0 / hsc;  // power of two: exact
  for (int i = tid; i < n; i += nt) {
    wr[i] *= ihsc;
    wi[i] *= ihsc;
  }
  if (tid == 0) {
    info[1] = nsweep;  // diagnostics: Francis sweeps, bulge steps
    info[2] = nstep;
    info[3] = (int)(cyc_chase >> 10);  // diagnostics: clock cycles / 1024 in the chase, in total
    info[4] = (int)((clock64() - cyc_all) >> 10);
#ifdef HQ_PROF
    info[5] = (int)(cyc_setup >> 10);  // sweep set-up to the first window, window transitions, last far update
    info[6] = (int)(cyc_trans >> 10);
    info[7] = (int)(cyc_last >> 10);
#endif
  }
}

// pick the nev largest |theta| (ties: Im descending, then lowest index; O23) and a split
// conjugate partner: nev+1 rounds of a block-wide arg-max over the unused eigenvalues
__device__ __forceinline__ bool sel_better(double m1, double i1, int k1, double m2, double i2, int k2) {
  if (k2 < 0) return k1 >= 0;
  if (k1 < 0) return false;
  if (m1 != m2) return m1 > m2;
  if (i1 != i2) return i1 > i2;
  return k1 < k2;
}

__global__ void __launch_bounds__(1024) select_kernel(const double* __restrict__ wr, const double* __restrict__ wi,
                                                      int n, int nev, int* __restrict__ sel, int* __restrict__ nsel,
                                                      double* __restrict__ th_re, double* __restrict__ th_im) {
  extern __shared__ int used[];  // n
  __shared__ double rm[32], ri[32];
  __shared__ int rk[32];
  __shared__ int cnt_s;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (blockDim.x + 31) >> 5;
  for (int i = tid; i < n; i += blockDim.x) used[i] = 0;
  if (tid == 0) cnt_s = 0;
  __syncthreads();
  const int want = min(nev, n);
  for (int c = 0; c < want + 1 && c < n; ++c) {
    double bm = -1.0, bi = 0.0;
    int bk = -1;
    for (int i = tid; i < n; i += blockDim.x) {
      if (used[i]) continue;
      const double mg = hypot(wr[i], wi[i]);
      if (sel_better(mg, wi[i], i, bm, bi, bk)) {
        bm = mg;
        bi = wi[i];
        bk = i;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double om = __shfl_xor_sync(0xffffffffu, bm, o), oi = __shfl_xor_sync(0xffffffffu, bi, o);
      const int ok = __shfl_xor_sync(0xffffffffu, bk, o);
      if (sel_better(om, oi, ok, bm, bi, bk)) {
        bm = om;
        bi = oi;
        bk = ok;
      }
    }
    if (lane == 0) {
      rm[wid] = bm;
      ri[wid] = bi;
      rk[wid] = bk;
    }
    __syncthreads();
    if (tid == 0) {
      for (int w = 1; w < nw; ++w)
        if (sel_better(rm[w], ri[w], rk[w], bm, bi, bk)) {
          bm = rm[w];
          bi = ri[w];
          bk = rk[w];
        }
      int cnt = cnt_s;
      if (c < want) {
        sel[cnt++] = bk;
        used[bk] = 1;
      } else {
        // position nev splits a conjugate pair?
        const int last = sel[cnt - 1];
        if (wi[last] != 0.0 && bk >= 0 && fabs(wr[bk] - wr[last]) <= 1e-12 * fabs(wr[last]) &&
            fabs(wi[bk] + wi[last]) <= 1e-12 * fabs(wi[last]))
          sel[cnt++] = bk;
      }
      cnt_s = cnt;
    }
    __syncthreads();
  }
  if (tid == 0) {
    const int cnt = cnt_s;
    *nsel = cnt;
    for (int t = 0; t < cnt; ++t) {
      th_re[t] = wr[sel[t]];
      th_im[t] = wi[sel[t]];
    }
  }
}

struct cplx {
  double r, i;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.r * b.r - a.i * b.i, a.r * b.i + a.i * b.r}; }
__device__ __forceinline__ cplx cdiv(cplx a, cplx b) {
  const double s = fabs(b.r) + fabs(b.i);
  const double ar = a.r / s, ai = a.i / s, br = b.r / s, bi = b.i / s;
  const double d = br * br + bi * bi;
  return {(ar * br + ai * bi) / d, (ai * br - ar * bi) / d};
}
__device__ __forceinline__ double cabs1(cplx a) { return fabs(a.r) + fabs(a.i); }

// One CTA per selected eigenvalue v: complex Hessenberg LU of (Mhat - theta I) with
// partial pivoting, then `iters` inverse-iteration solves.  Output y (d complex, unit
// 2-norm, largest-modulus entry real positive) in yr/yi[:, v] (ld = d).
__global__ void __launch_bounds__(256) inverse_iteration_kernel(const double* __restrict__ Mh, int d,
                                                                const double* __restrict__ th_re,
                                                                const double* __restrict__ th_im,
                                                                const int* __restrict__ nsel, double* __restrict__ work,
                                                                double* __restrict__ yr, double* __restrict__ yi,
                                                                int iters, double anorm) {
  const int v = blockIdx.x;
  if (v >= *nsel) return;
  extern __shared__ double smv[];
  cplx* b = reinterpret_cast<cplx*>(smv);  // d
  __shared__ double red[32];
  __shared__ cplx piv_l;
  __shared__ int swp;
  const int tid = threadIdx.x, nt = blockDim.x;
  // work layout: [A: nmax*d*d complex][L: nmax*d complex][perm: nmax*d int]
  const int64_t nmax = gridDim.x;
  cplx* A = reinterpret_cast<cplx*>(work) + (int64_t)v * d * d;  // column-major d x d
  cplx* L = reinterpret_cast<cplx*>(work) + nmax * d * d + (int64_t)v * d;
  int* perm = reinterpret_cast<int*>(reinterpret_cast<cplx*>(work) + nmax * d * d + nmax * d) + (int64_t)v * d;
  const cplx th = {th_re[v], th_im[v]};
  for (int64_t idx = tid; idx < (int64_t)d * d; idx += nt) {
    const int i = (int)(idx % d), j = (int)(idx / d);
    cplx e = {(i <= j + 1) ? Mh[idx] : 0.0, 0.0};
    if (i == j) {
      e.r -= th.r;
      e.i -= th.i;
    }
    A[idx] = e;
  }
  __syncthreads();
  double amax = 0.0;
  for (int64_t idx = tid; idx < (int64_t)d * d; idx += nt) amax = fmax(amax, cabs1(A[idx]));
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  if ((tid & 31) == 0) red[tid >> 5] = amax;
  __syncthreads();
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < (nt + 31) / 32; ++w) t = fmax(t, red[w]);
    red[0] = t;
  }
  __syncthreads();
  const double tiny = 1e-15 * fmax(anorm, red[0]) + 1e-300;
  __syncthreads();
  // LU: for k, pivot rows k / k+1, eliminate row k+1
  for (int k = 0; k < d - 1; ++k) {
    if (tid == 0) {
      cplx akk = A[k + (int64_t)k * d], ak1 = A[k + 1 + (int64_t)k * d];
      int s = cabs1(ak1) > cabs1(akk) ? 1 : 0;
      if (s) {
        cplx t = akk;
        akk = ak1;
        ak1 = t;
      }
      if (cabs1(akk) == 0.0) akk = {tiny, 0.0};
      swp = s;
      piv_l = cdiv(ak1, akk);
      perm[k] = s;
      L[k] = piv_l;
    }
    __syncthreads();
    const int s = swp;
    const cplx lk = piv_l;
    for (int j = k + tid; j < d; j += nt) {
      cplx r0 = A[k + (int64_t)j * d], r1 = A[k + 1 + (int64_t)j * d];
      if (s) {
        cplx t = r0;
        r0 = r1;
        r1 = t;
      }
      if (j == k && cabs1(r0) == 0.0) r0 = {tiny, 0.0};
      const cplx pr = cmul(lk, r0);
      r1.r -= pr.r;
      r1.i -= pr.i;
      A[k + (int64_t)j * d] = r0;
      A[k + 1 + (int64_t)j * d] = (j == k) ? cplx{0.0, 0.0} : r1;
    }
    __syncthreads();
  }
  if (tid == 0 && cabs1(A[(d - 1) + (int64_t)(d - 1) * d]) == 0.0) A[(d - 1) + (int64_t)(d - 1) * d] = {tiny, 0.0};
  for (int i = tid; i < d; i += nt) b[i] = {1.0 / (1.0 + 0.37 * (i % 11)), 0.0};
  __syncthreads();
  for (int it = 0; it < iters; ++it) {
    if (tid == 0) {
      // forward: apply P and L
      for (int k = 0; k < d - 1; ++k) {
        if (perm[k]) {
          cplx t = b[k];
          b[k] = b[k + 1];
          b[k + 1] = t;
        }
        const cplx pr = cmul(L[k], b[k]);
        b[k + 1].r -= pr.r;
        b[k + 1].i -= pr.i;
      }
    }
    __syncthreads();
    // backward: U y = b (column-oriented)
    for (int i = d - 1; i >= 0; --i) {
      if (tid == 0) b[i] = cdiv(b[i], A[i + (int64_t)i * d]);
      __syncthreads();
      const cplx yi_ = b[i];
      for (int l = tid; l < i; l += nt) {
        const cplx pr = cmul(A[l + (int64_t)i * d], yi_);
        b[l].r -= pr.r;
        b[l].i -= pr.i;
      }
      __syncthreads();
    }
    // normalise
    double loc = 0.0;
    for (int i = tid; i < d; i += nt) loc += b[i].r * b[i].r + b[i].i * b[i].i;
    const double nr = sqrt(block_sum(loc, red));
    for (int i = tid; i < d; i += nt) {
      b[i].r /= nr;
      b[i].i /= nr;
    }
    __syncthreads();
  }
  // canonical phase: largest-modulus entry real positive
  if (tid == 0) {
    int im = 0;
    double bm = -1.0;
    for (int i = 0; i < d; ++i) {
      const double mg = b[i].r * b[i].r + b[i].i * b[i].i;
      if (mg > bm) {
        bm = mg;
        im = i;
      }
    }
    const double mg = sqrt(bm);
    piv_l = {b[im].r / mg, -b[im].i / mg};  // conj phase
  }
  __syncthreads();
  const cplx ph = piv_l;
  for (int i = tid; i < d; i += nt) {
    const cplx z = cmul(b[i], ph);
    yr[i + (int64_t)v * d] = z.r;
    yi[i + (int64_t)v * d] = (th.i == 0.0) ? 0.0 : z.i;
  }
}

// ---- inverse iteration, pipelined: the same algorithm as inverse_iteration_kernel (Hessenberg LU of
// (Mhat - theta I) with partial pivoting between rows k and k+1, then `iters` solves), organised so that
// no step waits on an L2 round trip: the original rows of Mhat (strided in the column-major matrix) and
// the columns of U for the back substitution are staged into shared-memory rings by cp.async several
// steps ahead.  U is kept column-major in the work buffer.  One CTA per selected eigenvalue.
constexpr int II_T = 256;
constexpr int II_RING = 6;
__device__ __forceinline__ void ii_cp8(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void ii_cp16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void ii_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void ii_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

__global__ void __launch_bounds__(II_T) inverse_iteration_pipe_kernel(const double* __restrict__ Mh, int d,
                                                                      const double* __restrict__ th_re,
                                                                      const double* __restrict__ th_im,
                                                                      const int* __restrict__ nsel,
                                                                      double* __restrict__ work,
                                                                      double* __restrict__ yr,
                                                                      double* __restrict__ yi, int iters) {
  const int v = blockIdx.x;
  if (v >= *nsel) return;
  extern __shared__ __align__(16) double smi[];
  cplx* cur = reinterpret_cast<cplx*>(smi);       // d: the row carried through the elimination
  cplx* L = cur + d;                              // d: multipliers
  cplx* b = L + d;                                // d: solve vector
  cplx* cring = b + d;                            // II_RING x d: columns of U (back substitution)
  double* rring = reinterpret_cast<double*>(cring + (size_t)II_RING * d);  // II_RING x d: rows of Mhat
  int* perm = reinterpret_cast<int*>(rring + (size_t)II_RING * d);          // d
  __shared__ double red[32];
  __shared__ cplx piv_l, piv_p;
  __shared__ int swp;
  __shared__ double runmax;
  const int tid = threadIdx.x, nt = blockDim.x;
  cplx* U = reinterpret_cast<cplx*>(work) + (int64_t)v * d * d;  // column-major: U[l + i d], l <= i
  const cplx th = {th_re[v], th_im[v]};
  auto issue_row = [&](int r) {  // Mhat row r, columns r-1 .. d-1 (Hessenberg), into ring slot r % RING
    if (r < d) {
      double* dst = rring + (size_t)(r % II_RING) * d;
      for (int j = max(r - 1, 0) + tid; j < d; j += nt) ii_cp8(dst + j, Mh + r + (int64_t)j * d);
    }
    ii_commit();
  };
  // ring of RING slots, prefetch distance RING-1: rows 1..RING-1 now; iteration k issues row k+RING-1
  // into the slot of row k-1 (consumed in iteration k-1, free after this iteration's first barrier)
  for (int r = 1; r <= II_RING - 1; ++r) issue_row(r);
  for (int j = tid; j < d; j += nt) cur[j] = {Mh[(int64_t)j * d] - (j == 0 ? th.r : 0.0), j == 0 ? -th.i : 0.0};
  if (tid == 0) runmax = 0.0;
  // ---- LU: rows k (cur) and k+1 (Mhat row k+1 - theta e_{k+1}) compete for the pivot
  for (int k = 0; k < d - 1; ++k) {
    ii_wait<II_RING - 2>();  // row k+1 (group k+1 of RING-1+k) has landed (this thread's copies)
    __syncthreads();         // ... and everybody's; everybody is past iteration k-1
    issue_row(k + II_RING - 1);
    const double* nx = rring + (size_t)((k + 1) % II_RING) * d;
    if (tid == 0) {
      const cplx a = cur[k];
      const cplx bb = {nx[k], 0.0};  // column k of row k+1 (subdiagonal; theta sits on column k+1)
      runmax = fmax(runmax, fmax(cabs1(a), cabs1(bb)));
      const int sw = cabs1(bb) > cabs1(a) ? 1 : 0;
      cplx p = sw ? bb : a;
      const cplx o = sw ? a : bb;
      if (cabs1(p) == 0.0) p = {1e-15 * runmax + 1e-300, 0.0};
      swp = sw;
      piv_p = p;
      piv_l = cdiv(o, p);
      perm[k] = sw;
      L[k] = piv_l;
    }
    __syncthreads();
    const int sw = swp;
    const cplx lk = piv_l, pk = piv_p;
    for (int j = k + tid; j < d; j += nt) {
      const cplx cj = cur[j];
      const cplx nj = {nx[j] - (j == k + 1 ? th.r : 0.0), j == k + 1 ? -th.i : 0.0};
      const cplx pj = (j == k) ? pk : (sw ? nj : cj);
      const cplx oj = sw ? cj : nj;
      U[k + (int64_t)j * d] = pj;
      const cplx pr = cmul(lk, pj);
      cur[j] = {oj.r - pr.r, oj.i - pr.i};
    }
  }
  __syncthreads();
  if (tid == 0) {
    cplx p = cur[d - 1];
    if (cabs1(p) == 0.0) p = {1e-15 * runmax + 1e-300, 0.0};
    U[(d - 1) + (int64_t)(d - 1) * d] = p;
  }
  ii_wait<0>();
  __threadfence_block();
  __syncthreads();
  for (int i = tid; i < d; i += nt) b[i] = {1.0 / (1.0 + 0.37 * (i % 11)), 0.0};
  __syncthreads();
  auto issue_col = [&](int c) {  // column c of U (rows 0..c) into ring slot c % RING
    if (c >= 0) {
      cplx* dst = cring + (size_t)(c % II_RING) * d;
      for (int l = tid; l <= c; l += nt) ii_cp16(dst + l, U + l + (int64_t)c * d);
    }
    ii_commit();
  };
  for (int it = 0; it < iters; ++it) {
    for (int c = d - 1; c >= d - II_RING + 1; --c) issue_col(c);  // prefetch distance RING-1
    if (tid == 0) {  // forward: apply the row swaps and L
      for (int k = 0; k < d - 1; ++k) {
        if (perm[k]) {
          const cplx t = b[k];
          b[k] = b[k + 1];
          b[k + 1] = t;
        }
        const cplx pr = cmul(L[k], b[k]);
        b[k + 1].r -= pr.r;
        b[k + 1].i -= pr.i;
      }
    }
    // backward, column-oriented: y_i = b_i / U_ii, b_l -= U_li y_i (l < i)
    for (int i = d - 1; i >= 0; --i) {
      ii_wait<II_RING - 2>();  // column i landed (this thread's copies)
      __syncthreads();         // everybody's; b_i final; column i+1's slot is free
      issue_col(i - II_RING + 1);
      const cplx* col = cring + (size_t)(i % II_RING) * d;
      const cplx yi_ = cdiv(b[i], col[i]);
      __syncthreads();  // everybody has read b_i
      for (int l = tid; l < i; l += nt) {
        const cplx pr = cmul(col[l], yi_);
        b[l].r -= pr.r;
        b[l].i -= pr.i;
      }
      if (tid == 0) b[i] = yi_;
    }
    ii_wait<0>();
    __syncthreads();
    double loc = 0.0;
    for (int i = tid; i < d; i += nt) loc += b[i].r * b[i].r + b[i].i * b[i].i;
    const double nr = sqrt(block_sum(loc, red));
    for (int i = tid; i < d; i += nt) {
      b[i].r /= nr;
      b[i].i /= nr;
    }
    __syncthreads();
  }
  if (tid == 0) {  // canonical phase: largest-modulus entry real positive
    int im = 0;
    double bm = -1.0;
    for (int i = 0; i < d; ++i) {
      const double mg = b[i].r * b[i].r + b[i].i * b[i].i;
      if (mg > bm) {
        bm = mg;
        im = i;
      }
    }
    const double mg = sqrt(bm);
    piv_l = {b[im].r / mg, -b[im].i / mg};
  }
  __syncthreads();
  const cplx ph = piv_l;
  for (int i = tid; i < d; i += nt) {
    const cplx z = cmul(b[i], ph);
    yr[i + (int64_t)v * d] = z.r;
    yi[i + (int64_t)v * d] = (th.i == 0.0) ? 0.0 : z.i;
  }
}

// r_est[v] = ||D y - theta C y|| / ||C y||, D = SAB (s x d, col-major), C = SB
__global__ void srr_rest_kernel(const double* __restrict__ D, const double* __restrict__ C, int s, int d,
                                const double* __restrict__ yr, const double* __restrict__ yi,
                                const double* __restrict__ th_re, const double* __restrict__ th_im,
                                const int* __restrict__ nsel, double* __restrict__ rest) {
  const int v = blockIdx.x;
  if (v >= *nsel) return;
  __shared__ double red[64];
  const double a = th_re[v], b = th_im[v];
  double sr = 0.0, sc = 0.0;
  for (int q = threadIdx.x; q < s; q += blockDim.x) {
    double dr = 0, di = 0, cr = 0, ci = 0;
    for (int j = 0; j < d; ++j) {
      const double dd = D[q + (int64_t)j * s], cc = C[q + (int64_t)j * s];
      const double y0 = yr[j + (int64_t)v * d], y1 = yi[j + (int64_t)v * d];
      dr += dd * y0;
      di += dd * y1;
      cr += cc * y0;
      ci += cc * y1;
    }
    // D y - theta C y
    const double rr = dr - (a * cr - b * ci);
    const double ri = di - (a * ci + b * cr);
    sr += rr * rr + ri * ri;
    sc += cr * cr + ci * ci;
  }
  double t[2] = {sr, sc}, o[2];
  block_sum_n<2>(t, red, o);
  if (threadIdx.x == 0) rest[v] = sqrt(o[0]) / sqrt(o[1]);
}

// ------------------------------------------------------------------------------
cudaError_t launch_build_mhat(const double* H, int ldH, int d, const double* t, const double* gam, double* Mh,
                              cudaStream_t st) {
  build_mhat_kernel<<<(d * d + 255) / 256, 256, 0, st>>>(H, ldH, d, t, gam, Mh);
  return cudaGetLastError();
}
cudaError_t launch_hqr(double* a, int n, int lda, double* wr, double* wi, int* info, cudaStream_t st) {
  hqr_kernel<<<1, HQ_THREADS, 0, st>>>(a, n, lda, wr, wi, info);
  return cudaGetLastError();
}
cudaError_t launch_select(const double* wr, const double* wi, int n, int nev, int* sel, int* nsel, double* th_re,
                          double* th_im, cudaStream_t st) {
  select_kernel<<<1, 1024, sizeof(int) * n, st>>>(wr, wi, n, nev, sel, nsel, th_re, th_im);
  return cudaGetLastError();
}
size_t inverse_iteration_work_doubles(int d, int nmax) {
  return (size_t)nmax * d * d * 2 + (size_t)nmax * d * 2 + ((size_t)nmax * d + 1) / 2 + 16;
}
cudaError_t launch_inverse_iteration(const double* Mh, int d, const double* th_re, const double* th_im,
                                     const int* nsel, int nmax, double* work, double* yr, double* yi, int iters,
                                     double anorm, cudaStream_t st) {
  if (!getenv("SKS_II_OLD")) {  // pipelined version (default); SKS_II_OLD=1 for A/B
    const size_t smem = sizeof(double) * ((size_t)d * 2 * 3 + (size_t)II_RING * d * 2 + (size_t)II_RING * d) +
                        sizeof(int) * (size_t)d + 16;
    if (smem > 48 * 1024) {
      cudaError_t e = set_smem_attr(inverse_iteration_pipe_kernel, smem);
      if (e != cudaSuccess) return e;
    }
    (void)anorm;
    inverse_iteration_pipe_kernel<<<nmax, II_T, smem, st>>>(Mh, d, th_re, th_im, nsel, work, yr, yi, iters);
    return cudaGetLastError();
  }
  inverse_iteration_kernel<<<nmax, 256, sizeof(double) * 2 * d, st>>>(Mh, d, th_re, th_im, nsel, work, yr, yi,
                                                                       iters, anorm);
  return cudaGetLastError();
}
cudaError_t launch_srr_rest(const double* D, const double* C, int s, int d, const double* yr, const double* yi,
                            const double* th_re, const double* th_im, const int* nsel, int nmax, double* rest,
                            cudaStream_t st) {
  srr_rest_kernel<<<nmax, 256, 0, st>>>(D, C, s, d, yr, yi, th_re, th_im, nsel, rest);
  return cudaGetLastError();
}

}  // namespace sks
