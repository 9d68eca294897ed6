// stencil_ym.cu -- fused truncated-Arnoldi step for the 2D 5-point operator, y-march design.
//
// The 2D counterpart of stencil_zm.cu (same arithmetic: Eq. partorth, Alg. 1
// P:1300-1307; one launch forms w_j and the next step's partial sums).  A CTA owns an x-segment of
// YX = 252 output columns and marches through a range of y lines, ZS lines per step:
//
//   * per step the TMA brings ZS+2 lines of U (256 wide: 2-point x halo) and ZS lines of each window
//     vector V_l into one of two stages (mbarrier completion, out-of-bounds x zero-filled: the
//     Dirichlet x boundary costs nothing);
//   * each of the 254 W-segment threads owns one x column: the y neighbours of the 5-point stencil
//     come from the march (registers), only the x neighbours from shared memory -- 3 shared loads per
//     point for w_j, 2 for A w_j (the tiled 2D kernel loads all 4 neighbours and recomputes a 2D halo);
//   * after ONE __syncthreads per step, interior threads form A w_j for the ZS lines one behind, store
//     w_j and accumulate ||w||^2, <w,Aw>, ||Aw||^2 and the window dots in registers;
//   * several CTAs per SM (64 KB of shared memory each at k = 2).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "internal.h"
#include "step.cuh"
#include "tma.cuh"

namespace sks {

constexpr int YX = 252;         // output columns per tile
constexpr int YWX = YX + 2;     // W segment (1-point x halo for A w_j)
constexpr int YUX = YX + 4;     // U / V line box (2-point halo; TMA box dimension <= 256)
constexpr int YT = 256;         // threads (254 W columns + 2 idle)
constexpr int YCPS = 2;         // resident CTAs per SM (register budget: 128 per thread)

constexpr int YM_MAXG = 2 * 148;  // CTAs covered by the partition table
struct YmArgs {
  int ucol;
  int vcol[SKS_KMAX];
  int tiles_x;
  int64_t units;  // tiles_x * nz
  int nv;
  int use_ub;     // 1: CTA b owns units [ub[b], ub[b+1]) (step-balanced partition), else proportional
  int32_t ub[YM_MAXG + 1];
};

__host__ __device__ constexpr int ym_al16(int d) { return (d + 15) & ~15; }
template <int KM, int ZS>
__host__ __device__ constexpr int ym_ublk() { return ym_al16(YUX * (ZS + 2)); }
template <int KM, int ZS>
__host__ __device__ constexpr int ym_vblk() { return ym_al16(YUX * ZS); }
template <int KM, int ZS>
__host__ __device__ constexpr int ym_stage() { return ym_ublk<KM, ZS>() + (KM - 1) * ym_vblk<KM, ZS>(); }
template <int KM, int ZS>
__host__ __device__ constexpr size_t ym_smem_bytes() {
  return 128 + sizeof(double) * ((size_t)2 * ym_stage<KM, ZS>() + (size_t)(3 * ZS) * YWX);
}

// FE (k <= 2, default; SKS_YM_FE=0 for A/B): forward-edge form of the next step's quadratic form and <A^T U, w_j>
// in phase A, as in the 3D pair kernel (stencil_zm.cu, reading O39): phase B reads only the +x neighbour from the ring
// (+y is the next line, in registers) and forms no A w_j.
template <int KM, int ZS, bool FULL, bool USL, bool FE = false>
__global__ void __launch_bounds__(YT, YCPS)
    step2d_ym_kernel(StepArgs a, YmArgs z, const __grid_constant__ CUtensorMap tmU,
                     const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smraw_y[];
  double* sm = reinterpret_cast<double*>(smraw_y + ((128u - (smem_u32(smraw_y) & 127u)) & 127u));
  constexpr int STG = ym_stage<KM, ZS>();
  constexpr int UB = ym_ublk<KM, ZS>(), VB = ym_vblk<KM, ZS>();
  constexpr int R = 3 * ZS;  // w_j line ring
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
  pdl_wait_and_release();                   // programmatic dependent launch (see stencil_zm.cu)
  const int nv = FULL ? KM - 1 : z.nv;      // = cf.nv (host-known)
  const uint32_t sbytes = (uint32_t)(YUX * (ZS + 2) * 8 + nv * YUX * ZS * 8);
  const int m = (int)a.m, nz = (int)a.nz, z0g = (int)a.z0, G = a.G;
  const int64_t u_lo = z.use_ub ? (int64_t)z.ub[blockIdx.x] : (z.units * blockIdx.x) / gridDim.x;
  const int64_t u_hi = z.use_ub ? (int64_t)z.ub[blockIdx.x + 1] : (z.units * (blockIdx.x + 1)) / gridDim.x;
  // the first piece's first two stages go out before the prologue's partials reduction
  int pre = 0;
  if (tid == 0 && u_lo < u_hi) {
    const int col = (int)(u_lo / nz), za = (int)(u_lo % nz);
    const int64_t zr = za + (u_hi - u_lo);
    const int zb = (int)(zr < nz ? zr : nz);
    const int x0 = col * YX, wa = za - 1;
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;
    for (int t = 0; t < 2 && t < nsteps; ++t) {
      double* dst = sm + t * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[t], sbytes);
      tma_load_3d(dst, &tmU, &bar[t], x0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_3d(dst + UB + l * VB, &tmV, &bar[t], x0 - 2, p0 + G, z.vcol[l]);
      pre = t + 1;
    }
  }
  if (!step_prologue(a, &cf, red)) {  // contains __syncthreads
    for (int t = 0; t < pre; ++t) mbar_wait(&bar[t], 0u);  // no bulk copy may outlive the CTA
    return;
  }
  const int64_t pl = a.plane;  // = m (a line)
  const double cc = a.cc, cm = a.cm, cp = a.cp, alpha = cf.alpha, beta_u = cf.beta_u;
  double cl[KM - 1];
#pragma unroll
  for (int l = 0; l < KM - 1; ++l) cl[l] = (l < nv) ? cf.c[l] : 0.0;
  constexpr bool uslot = USL;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;

  const int bx = tid;                   // W-segment column (x0 - 1 + bx)
  const bool wt = bx < YWX;
  const int cu = bx + 1;                // U/V line offset (box origin x0 - 2)
  const bool inner = bx >= 1 && bx <= YX;

  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;

  uint32_t phase = 0;
  uint32_t sidx = 0;
  bool first = true;
  for (int64_t u = u_lo; u < u_hi;) {
    const int col = (int)(u / nz);
    const int za = (int)(u % nz);
    const int64_t zr = za + (u_hi - u);
    const int zb = (int)(zr < nz ? zr : nz);
    u += zb - za;
    const int x0 = col * YX;
    const int wa = za - 1;                           // first w_j line of the piece
    const int nsteps = (zb - wa + 1 + ZS - 1) / ZS;  // w_j lines wa .. zb
    const uint32_t s0 = sidx;
    auto issue = [&](int t) {  // stage t: U lines [wa+t ZS-1, wa+t ZS+ZS], V lines [wa+t ZS, +ZS)
      const uint32_t slot = (s0 + (uint32_t)t) & 1u;
      double* dst = sm + slot * STG;
      const int p0 = wa + t * ZS;
      mbar_arrive_expect_tx(&bar[slot], sbytes);
      tma_load_3d(dst, &tmU, &bar[slot], x0 - 2, p0 - 1 + G, z.ucol);
      for (int l = 0; l < nv; ++l) tma_load_3d(dst + UB + l * VB, &tmV, &bar[slot], x0 - 2, p0 + G, z.vcol[l]);
    };
    if (tid == 0 && !first) {
      issue(0);
      if (nsteps > 1) issue(1);
    }
    first = false;
    double wp1 = 0.0, wp2 = 0.0;
    double vlast[KM - 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) vlast[l] = 0.0;
    const int gxw = x0 - 1 + bx;
    const bool xin = wt && (unsigned)gxw < (unsigned)m;
    const bool aw = inner && gxw < m;
    double* wcol = Wout + (int64_t)(wa - 1) * pl + gxw;  // line wa-1 of the column
    const double am = xin ? alpha : 0.0, bm = xin ? beta_u : 0.0;
    double clm[KM - 1];
#pragma unroll
    for (int l = 0; l < KM - 1; ++l) clm[l] = xin ? cl[l] : 0.0;
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
      const bool fast = t >= T0 && p0 + ZS - 1 <= zb && z0g + p0 + ZS - 1 < m;
      double w[ZS], c[ZS + 2], v[KM - 1][ZS];
      double* rw = ring + SBW * YWX + bx;
      const double* rp = ring + SBP * YWX + bx;
#pragma unroll
      for (int k = 0; k < ZS + 2; ++k) c[k] = sU[k * YUX + cu];
#pragma unroll
      for (int i = 0; i < ZS; ++i) {
        const int p = p0 + i;
#pragma unroll
        for (int l = 0; l < KM - 1; ++l) v[l][i] = (FULL || l < nv) ? sV[l * VB + i * YUX + cu] : 0.0;
        const double* q = sU + (i + 1) * YUX + cu;
        const double smn = q[-1] + c[i], spl = q[1] + c[i + 2];
        const double Au = cc * c[i + 1] + cm * smn + cp * spl;
        double wv;
        if (fast) {
          wv = am * Au + bm * c[i + 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (FULL || l < nv) wv += clm[l] * v[l][i];
        } else {
          wv = alpha * Au + beta_u * c[i + 1];
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (FULL || l < nv) wv += cl[l] * v[l][i];
          wv = (xin && (unsigned)(z0g + p) < (unsigned)m && p <= zb) ? wv : 0.0;
        }
        w[i] = wv;
        if (wt) rw[i * YWX] = wv;
        if constexpr (FE && USL) {  // <U, A w_j> = <A^T U, w_j> on the owned points (line p in [za, zb))
          const double ta = (aw && p >= za && p < zb) ? cc * c[i + 1] + cp * smn + cm * spl : 0.0;
          acc[KM + 2] += ta * wv;
        }
      }
      __syncthreads();
      if (tid == 0 && t + 2 < nsteps) issue(t + 2);
      if (aw) {
        double* wo = wcol;
#pragma unroll
        for (int i = 0; i < ZS; ++i) {
          const int qp = p0 - 1 + i;
          if (fast || (qp >= za && qp < zb)) {
            const double wq = (i == 0) ? wp1 : w[i - 1];
            const double wqm = (i == 0) ? wp2 : (i == 1 ? wp1 : w[i - 2]);
            const double* r = (i == 0) ? rp : rw + (i - 1) * YWX;
            if constexpr (FE) {  // forward edges: +x from the ring, +y = the next line
              *wo = wq;
              acc[0] += wq * wq;
              acc[2] += wq * (r[1] + w[i]);
              (void)wqm;
              wo += pl;
              continue;
            }
            const double Aw = cc * wq + cm * (r[-1] + wqm) + cp * (r[1] + w[i]);
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
    __syncthreads();
  }
  if constexpr (FE) {  // slot 1: <w, A w> = cc ||w||^2 + (cm + cp) sum of forward-edge products; no ||A w||^2
    acc[1] = cc * acc[0] + (cm + cp) * acc[2];
    acc[2] = 0.0;
  }
  step_epilogue<KM>(a, &cf, acc, red);
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_enc_ym = nullptr;

static bool ym_encode_fn() {
  if (g_enc_ym) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_enc_ym = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// 3D map {x: m, line_storage: nz+2G, column: ncol} over columns of pitch ld
static bool ym_encode(CUtensorMap* out, const double* base, int64_t m, int64_t nz, int G, int64_t ld, int64_t ncol,
                      int lines) {
  if (!ym_encode_fn()) return false;
  cuuint64_t dims[3] = {(cuuint64_t)m, (cuuint64_t)(nz + 2 * G), (cuuint64_t)ncol};
  cuuint64_t strides[2] = {(cuuint64_t)(m * 8), (cuuint64_t)(ld * 8)};
  cuuint32_t box[3] = {(cuuint32_t)YUX, (cuuint32_t)lines, 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = g_enc_ym(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct YmMaps {
  CUtensorMap WU, WV, XU, FV, VU;
  MapKey key[5];
  int64_t part_key = -1;  // step-balanced partition cache
  bool part_ok = false;
  int32_t ub[YM_MAXG + 1];
};

template <int KM>
constexpr int ym_zs() {
  return ym_smem_bytes<KM, 4>() <= 226 * 1024 / YCPS - 1024 ? 4 : 2;
}

bool stencil_ym_supported(int dim, int64_t m, int k) {
  // TMA global strides must be multiples of 16 bytes; on small grids (C2: m = 512, 2 MB vectors) the
  // launch is latency-bound and the tiled 2D kernel's shorter pipeline wins (44.2 vs 49.6 ms)
  if (dim != 2 || m % 2 || m < 1024) return false;
  const char* e = getenv("SKS_NO_YM");
  if (e && e[0] == '1') return false;
  return ym_encode_fn();
}

void stencil_ym_tiling(int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid) {
  a->tiles_x = (int)((m + YX - 1) / YX);
  a->tiles_y = 1;
  a->zchunk = 0;
  a->ntiles = (int64_t)a->tiles_x * nz;  // (segment, line) units
  *grid = (int)std::max<int64_t>(1, std::min<int64_t>(a->ntiles, (int64_t)num_sms * YCPS));
}

template <int KM, bool FULL, bool USL>
static cudaError_t ym_launch_v(const StepArgs& a, const YmArgs& z, const CUtensorMap& mu, const CUtensorMap& mv,
                               int grid, cudaStream_t st) {
  constexpr int ZS = ym_zs<KM>();
  const size_t smem = ym_smem_bytes<KM, ZS>();
  if constexpr (KM == 2) {
    static int fe = -1;
    if (fe < 0) {
      const char* e = getenv("SKS_YM_FE");
      fe = e ? (e[0] == '1') : 1;
    }
    if (fe) {
      StepArgs af = a;
      af.fe = 1;
      if (cudaError_t e = set_smem_attr(step2d_ym_kernel<KM, ZS, FULL, USL, true>, smem)) return e;
      return launch_pdl(step2d_ym_kernel<KM, ZS, FULL, USL, true>, grid, YT, smem, st, af, z, mu, mv);
    }
  }
  if (cudaError_t e = set_smem_attr(step2d_ym_kernel<KM, ZS, FULL, USL>, smem)) return e;
  return launch_pdl(step2d_ym_kernel<KM, ZS, FULL, USL>, grid, YT, smem, st, a, z, mu, mv);
}

template <int KM>
static cudaError_t ym_launch(const StepArgs& a, const YmArgs& z, const CUtensorMap& mu, const CUtensorMap& mv,
                             int grid, cudaStream_t st) {
  const bool full = z.nv == KM - 1;
  const bool usl = a.mode == 0 && a.k >= 2;
  if (full && usl) return ym_launch_v<KM, true, true>(a, z, mu, mv, grid, st);
  if (full) return ym_launch_v<KM, true, false>(a, z, mu, mv, grid, st);
  if (usl) return ym_launch_v<KM, false, true>(a, z, mu, mv, grid, st);
  return ym_launch_v<KM, false, false>(a, z, mu, mv, grid, st);
}

// mode 0: U = column j-1, V_l = columns lo+l of W; mode 1: U = x, V0 = f; mode 2: U = v0.
cudaError_t launch_step_stencil_ym(const StepArgs& a, const double* W, int64_t ncol, const double* xb,
                                   const double* fb, const double* vb, int grid, cudaStream_t st, void** cache) {
  YmMaps* mp = reinterpret_cast<YmMaps*>(*cache);
  if (!mp) {
    mp = new YmMaps();
    *cache = mp;
  }
  const int km = step_km(a.k);
  const int zs = km == 2 ? ym_zs<2>() : (km == 4 ? ym_zs<4>() : ym_zs<8>());
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
    if (!ym_encode(mpp, base, a.m, a.nz, a.G, a.ld, nc, ub ? zs + 2 : zs)) return false;
    mp->key[slot] = key;
    return true;
  };
  YmArgs z;
  memset(&z, 0, sizeof(z));
  z.tiles_x = a.tiles_x;
  z.units = a.ntiles;
  z.nv = (a.mode == 0) ? std::min(a.j, a.k) - 1 : (a.mode == 1 ? 1 : 0);
  {  // step-balanced partition (stencil_zm.cu), cached per (units, nz, grid, zs)
    static int bal = -1;
    if (bal < 0) {
      const char* e = getenv("SKS_ZM_BALANCE");
      bal = e ? (e[0] == '1') : 1;
    }
    if (bal) {
      const int64_t pk = z.units * 1000003 + a.nz * 131 + grid * 7 + zs;
      if (mp->part_key != pk) {
        mp->part_ok = step_partition(z.units, a.nz, grid, zs, YM_MAXG, mp->ub);
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
    case 2: return ym_launch<2>(a, z, *mu, *mv, grid, st);
    case 4: return ym_launch<4>(a, z, *mu, *mv, grid, st);
    default: return ym_launch<8>(a, z, *mu, *mv, grid, st);
  }
}

void stencil_ym_free(void* cache) { delete reinterpret_cast<YmMaps*>(cache); }

}  // namespace sks
