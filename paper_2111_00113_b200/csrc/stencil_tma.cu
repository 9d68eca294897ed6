// stencil_tma.cu -- fused truncated-Arnoldi step, TMA-fed (sm_100a), for even m.
//
// Same arithmetic as stencil.cu (see step.cuh), different data movement:
//   * all basis columns are one 4D (3D grid) / 3D (2D grid) tensor map
//     {x, y, z_storage, column}; a tile's U box (2-point halo) and window-vector boxes
//     (1-point halo) arrive by cp.async.bulk.tensor with out-of-bounds ZERO fill, so
//     the Dirichlet x/y boundary costs nothing and no thread does address arithmetic;
//   * persistent CTAs (one or two per SM) walk the tiles; a 2-stage mbarrier pipeline
//     prefetches tile t+1 while tile t is computed;
//   * 3D: each thread marches along z through its (x,y) column, keeping the z-neighbours
//     of U and of w_j in registers (5 shared loads per 7-point stencil instead of 7).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>

#include "common.cuh"
#include "internal.h"
#include "step.cuh"
#include "tma.cuh"

namespace sks {

struct TmaCols {
  int ucol;
  int vcol[SKS_KMAX];
  int nv;  // window vectors of this launch (= StepCoef::nv, known on the host)
};

// ---------------------------------------------------------------- 3D
constexpr int Q3X = 32, Q3Y = 8, Q3Z = 8;                    // outputs per tile
constexpr int QU3X = Q3X + 4, QU3Y = Q3Y + 4, QU3Z = Q3Z + 4;  // U box 36 x 12 x 12
constexpr int QV3X = Q3X + 2, QV3Y = Q3Y + 2, QV3Z = Q3Z + 2;  // W box 34 x 10 x 10
constexpr int QU3 = QU3X * QU3Y * QU3Z;                       // 5184
constexpr int QV3 = QV3X * QV3Y * QV3Z;                       // 3400 (W box)
constexpr int QV3P = 3408;                                    // W box padded to 128 B
// window-vector (V) boxes start at x0-2 like U: the TMA box origin's innermost byte
// offset must be 16-byte aligned (odd fp64 x-coordinates fault), so V is 36 wide.
constexpr int QB3X = QU3X;                                    // 36
constexpr int QB3 = QB3X * QV3Y * QV3Z;                       // 3600 (= 225 x 128 B)
constexpr int QT = 512;                                       // threads

template <int KM, int NST>
__global__ void __launch_bounds__(QT, 1)
    step3d_tma_kernel(StepArgs a, TmaCols tc, const __grid_constant__ CUtensorMap tmU,
                      const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smraw_t[];
  // align to 128 B by offsetting the shared array itself (keeps the pointer in the shared
  // window so the compiler emits LDS/STS, not generic loads)
  double* smt = reinterpret_cast<double*>(smraw_t + ((128u - (smem_u32(smraw_t) & 127u)) & 127u));
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ __align__(8) uint64_t bar[NST];
  const int tid = threadIdx.x;
  if (tid == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  pdl_wait_and_release();                   // programmatic dependent launch (see stencil_zm.cu)
  if (!step_prologue(a, &cf, red)) return;  // contains __syncthreads
  constexpr int STAGE = QU3 + (KM - 1) * QB3;
  double* sW = smt + NST * STAGE;
  const int nv = cf.nv;
  const uint32_t bytes = (uint32_t)(QU3 * 8 + nv * QB3 * 8);
  const int64_t m = a.m, nz = a.nz, pl = a.plane;
  const int G = a.G;
  const double cc = a.cc, cm = a.cm, cp = a.cp, alpha = cf.alpha, beta_u = cf.beta_u;
  double cl[KM - 1];
#pragma unroll
  for (int l = 0; l < KM - 1; ++l) cl[l] = (l < nv) ? cf.c[l] : 0.0;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;
  const unsigned ntx = (unsigned)a.tiles_x, nty = (unsigned)a.tiles_y;
  const int ntiles = (int)a.ntiles;
  const int mi = (int)m, nzi = (int)nz, z0g = (int)a.z0;
  __shared__ int tco[NST][3];  // tile coordinates of each stage (written by the issuing thread)

  auto issue = [&](int tile, int s) {
    const unsigned t = (unsigned)tile;
    const int tx = (int)(t % ntx);
    const unsigned r = t / ntx;
    const int ty = (int)(r % nty), tz = (int)(r / nty);
    tco[s][0] = tx * Q3X;
    tco[s][1] = ty * Q3Y;
    tco[s][2] = tz * Q3Z;
    double* base = smt + s * STAGE;
    mbar_arrive_expect_tx(&bar[s], bytes);  // release: tco[s] is visible to the waiters
    tma_load_4d(base, &tmU, &bar[s], tx * Q3X - 2, ty * Q3Y - 2, tz * Q3Z - 2 + G, tc.ucol);
    for (int l = 0; l < nv; ++l)
      tma_load_4d(base + QU3 + l * QB3, &tmV, &bar[s], tx * Q3X - 2, ty * Q3Y - 1, tz * Q3Z - 1 + G, tc.vcol[l]);
  };

  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;

  // per-thread constants of the two phases
  const bool wthr = tid < QV3X * QV3Y;
  const int xw = tid % QV3X, yw = tid / QV3X;
  const int cu = (yw + 1) * QU3X + xw + 1;   // U-box (x,y) offset of this W column
  const int cv = yw * QB3X + xw + 1;          // V-box (x,y) offset of this W column
  const int cx = tid & 31, cy = (tid >> 5) & 7, zh = tid >> 8;
  const int cw = (cy + 1) * QV3X + cx + 1;    // W-box (x,y) offset of this output column
  const int cuo = (cy + 2) * QU3X + cx + 2;   // U-box offset of this output column
  const int cvo = (cy + 1) * QB3X + cx + 2;   // V-box offset of this output column

  const int first = blockIdx.x, stride = gridDim.x;
  if (tid == 0 && first < ntiles) issue(first, 0);
  int it = 0;
  for (int tile = first; tile < ntiles; tile += stride, ++it) {
    const int s = (NST == 2) ? (it & 1) : 0;
    if (NST == 2 && tid == 0 && tile + stride < ntiles) issue(tile + stride, s ^ 1);
    const double* sU = smt + s * STAGE;
    const double* sV = sU + QU3;
    mbar_wait(&bar[s], (uint32_t)((NST == 2 ? (it >> 1) : it) & 1));
    const int x0 = tco[s][0], y0 = tco[s][1], zt0 = tco[s][2];
    // ---- W = alpha A U + beta_u U + sum c_l V_l on the 34 x 10 x 10 box (zero outside the domain)
    if (wthr) {
      const int gx = x0 - 1 + xw, gy = y0 - 1 + yw;
      const bool colin = (unsigned)gx < (unsigned)mi && (unsigned)gy < (unsigned)mi;
      const int gz0 = z0g + zt0 - 1;
      double um = sU[cu];
      double u0 = sU[QU3X * QU3Y + cu];
#pragma unroll
      for (int zw = 0; zw < QV3Z; ++zw) {
        const double* p1 = sU + (zw + 1) * QU3X * QU3Y + cu;
        const double up = sU[(zw + 2) * QU3X * QU3Y + cu];
        double w = 0.0;
        if (colin && (unsigned)(gz0 + zw) < (unsigned)mi) {
          const double Au = cc * u0 + cm * (p1[-1] + p1[-QU3X] + um) + cp * (p1[1] + p1[QU3X] + up);
          w = alpha * Au + beta_u * u0;
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (l < nv) w += cl[l] * sV[l * QB3 + zw * QB3X * QV3Y + cv];
        }
        sW[zw * QV3X * QV3Y + yw * QV3X + xw] = w;
        um = u0;
        u0 = up;
      }
    }
    __syncthreads();
    // ---- A w_j, dots and the store on the 32 x 8 x 8 output box (two z-halves)
    {
      const bool xyin = (x0 + cx < mi) && (y0 + cy < mi);
      double* wo = Wout + (int64_t)(zt0 + zh * 4) * pl + (int64_t)(y0 + cy) * m + x0 + cx;
      double wm = sW[(zh * 4) * QV3X * QV3Y + cw];
      double w0 = sW[(zh * 4 + 1) * QV3X * QV3Y + cw];
#pragma unroll
      for (int zz = 0; zz < 4; ++zz) {
        const int z = zh * 4 + zz;
        const double* q1 = sW + (z + 1) * QV3X * QV3Y + cw;
        const double wp = sW[(z + 2) * QV3X * QV3Y + cw];
        if (xyin && zt0 + z < nzi) {
          const double Aw = cc * w0 + cm * (q1[-1] + q1[-QV3X] + wm) + cp * (q1[1] + q1[QV3X] + wp);
          *wo = w0;
          acc[0] += w0 * w0;
          acc[1] += w0 * Aw;
          acc[2] += Aw * Aw;
          if (cf.uslot >= 0) acc[KM + 2] += sU[(z + 2) * QU3X * QU3Y + cuo] * Aw;
#pragma unroll
          for (int l = 0; l < KM - 1; ++l)
            if (l < nv) acc[3 + l] += sV[l * QB3 + (z + 1) * QB3X * QV3Y + cvo] * Aw;
        }
        wo += pl;
        wm = w0;
        w0 = wp;
      }
    }
    __syncthreads();
    if (NST == 1 && tid == 0 && tile + stride < ntiles) issue(tile + stride, 0);
  }
  step_epilogue<KM>(a, &cf, acc, red);
}

// ---------------------------------------------------------------- 2D
#ifndef Q2Y_M
#define Q2Y_M 32  // 2D tile height (C2: 64 x 32 -> 128 tiles)
#endif
#ifndef Q2_MINB
#define Q2_MINB 1  // resident CTAs per SM the 2D kernel is compiled for
#endif
constexpr int Q2X = 64, Q2Y = Q2Y_M;
constexpr int QU2X = Q2X + 4, QU2Y = Q2Y + 4;  // 68 x 36
constexpr int QV2X = Q2X + 2, QV2Y = Q2Y + 2;  // 66 x 34
constexpr int QU2 = QU2X * QU2Y;               // 2448
constexpr int QV2 = QV2X * QV2Y;               // 2244 (W box)
constexpr int QV2P = (QV2 + 15) / 16 * 16;       // W box padded to 128 B (2256 at 64 x 32)
constexpr int QB2X = QU2X;                     // V box 68 wide (16-byte aligned origin, see 3D)
constexpr int QB2 = QB2X * QV2Y;               // 2312
constexpr int QB2P = (QB2 + 15) / 16 * 16;       // 2320 at 64 x 32

template <int KM, int NST>
__global__ void __launch_bounds__(QT, Q2_MINB)
    step2d_tma_kernel(StepArgs a, TmaCols tc, const __grid_constant__ CUtensorMap tmU,
                      const __grid_constant__ CUtensorMap tmV) {
  extern __shared__ __align__(128) unsigned char smraw_t[];
  // align to 128 B by offsetting the shared array itself (keeps the pointer in the shared
  // window so the compiler emits LDS/STS, not generic loads)
  double* smt = reinterpret_cast<double*>(smraw_t + ((128u - (smem_u32(smraw_t) & 127u)) & 127u));
  __shared__ StepCoef cf;
  __shared__ double red[SKS_NP * 32];
  __shared__ __align__(8) uint64_t bar[NST];
  const int tid = threadIdx.x;
  if (tid == 0) {
    tma_prefetch_desc(&tmU);
    tma_prefetch_desc(&tmV);
    for (int s = 0; s < NST; ++s) mbar_init(&bar[s], 1);
    fence_mbar_init();
  }
  pdl_wait_and_release();
  constexpr int STAGE = QU2 + (KM - 1) * QB2P;
  double* sW = smt + NST * STAGE;
  const int nv = tc.nv;  // = cf.nv: the first tiles' loads go out before the prologue's reduction
  const uint32_t bytes = (uint32_t)(QU2 * 8 + nv * QB2 * 8);
  const int ntx = a.tiles_x;
  const int64_t ntiles = a.ntiles;
  const int G = a.G;
  auto issue = [&](int64_t tile, int s) {
    const int tx = (int)(tile % ntx);
    const int ty = (int)(tile / ntx);
    double* base = smt + s * STAGE;
    mbar_arrive_expect_tx(&bar[s], bytes);
    tma_load_3d(base, &tmU, &bar[s], tx * Q2X - 2, ty * Q2Y - 2 + G, tc.ucol);
    for (int l = 0; l < nv; ++l)
      tma_load_3d(base + QU2 + l * QB2P, &tmV, &bar[s], tx * Q2X - 2, ty * Q2Y - 1 + G, tc.vcol[l]);
  };
  const int64_t first = blockIdx.x, stride = gridDim.x;
  int pre = 0;
  if (tid == 0 && first < ntiles) {
    issue(first, 0);
    pre = 1;
    if (NST == 2 && first + stride < ntiles) {
      issue(first + stride, 1);
      pre = 2;
    }
  }
  if (!step_prologue(a, &cf, red)) {
    for (int s = 0; s < pre; ++s) mbar_wait(&bar[s], 0u);  // no bulk copy may outlive the CTA
    return;
  }
  const int64_t m = a.m, nz = a.nz;
  const double cc = a.cc, cm = a.cm, cp = a.cp, alpha = cf.alpha, beta_u = cf.beta_u;
  double cl[KM - 1];
#pragma unroll
  for (int l = 0; l < KM - 1; ++l) cl[l] = (l < nv) ? cf.c[l] : 0.0;
  double* Wout = a.W + (a.mode == 0 ? (int64_t)a.j * a.ld : 0) + a.off;

  double acc[KM + 3];
#pragma unroll
  for (int i = 0; i < KM + 3; ++i) acc[i] = 0.0;
  int it = 0;
  for (int64_t tile = first; tile < ntiles; tile += stride, ++it) {
    const int s = (NST == 2) ? (it & 1) : 0;
    if (NST == 2 && tid == 0 && it >= 1 && tile + stride < ntiles) issue(tile + stride, s ^ 1);
    const int64_t x0 = (tile % ntx) * Q2X, yt0 = (tile / ntx) * Q2Y;
    const double* sU = smt + s * STAGE;
    const double* sV = sU + QU2;
    mbar_wait(&bar[s], (uint32_t)((NST == 2 ? (it >> 1) : it) & 1));
    for (int p = tid; p < QV2; p += QT) {
      const int xw = p % QV2X, yw = p / QV2X;
      const int64_t gx = x0 - 1 + xw, gy = a.z0 + yt0 - 1 + yw;
      double w = 0.0;
      if (gx >= 0 && gx < m && gy >= 0 && gy < m) {
        const double* c = sU + (yw + 1) * QU2X + xw + 1;
        const double u = c[0];
        const double Au = cc * u + cm * (c[-1] + c[-QU2X]) + cp * (c[1] + c[QU2X]);
        w = alpha * Au + beta_u * u;
#pragma unroll
        for (int l = 0; l < KM - 1; ++l)
          if (l < nv) w += cl[l] * sV[l * QB2P + yw * QB2X + xw + 1];
      }
      sW[p] = w;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < (Q2X * Q2Y) / QT; ++i) {
      const int p = tid + i * QT;
      const int x = p & (Q2X - 1), y = p / Q2X;
      if (x0 + x < m && yt0 + y < nz) {
        const double* c = sW + (y + 1) * QV2X + x + 1;
        const double w = c[0];
        const double Aw = cc * w + cm * (c[-1] + c[-QV2X]) + cp * (c[1] + c[QV2X]);
        Wout[(yt0 + y) * m + x0 + x] = w;
        acc[0] += w * w;
        acc[1] += w * Aw;
        acc[2] += Aw * Aw;
        if (cf.uslot >= 0) acc[KM + 2] += sU[(y + 2) * QU2X + x + 2] * Aw;
#pragma unroll
        for (int l = 0; l < KM - 1; ++l)
          if (l < nv) acc[3 + l] += sV[l * QB2P + (y + 1) * QB2X + x + 2] * Aw;
      }
    }
    __syncthreads();
    if (NST == 1 && tid == 0 && tile + stride < ntiles) issue(tile + stride, 0);
  }
  step_epilogue<KM>(a, &cf, acc, red);
}

// ---------------------------------------------------------------- host side
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool get_encode() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess || !fn) {
    cudaGetLastError();
    return false;
  }
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

// map over `ncol` columns (pitch ld doubles) of a ghost-layout vector set starting at `base`
// 3D grid: dims {m, m, nz+2G, ncol}; 2D grid: dims {m, nz+2G, ncol}.  box = U (halo 2) or V (halo 1).
static bool encode_map(CUtensorMap* out, int dim, const double* base, int64_t m, int64_t nz, int G, int64_t ld,
                       int64_t ncol, bool ubox) {
  if (!get_encode()) return false;
  cuuint64_t dims[4], strides[3];
  cuuint32_t box[4], es[4] = {1, 1, 1, 1};
  cuuint32_t rank;
  if (dim == 3) {
    rank = 4;
    dims[0] = m; dims[1] = m; dims[2] = nz + 2 * G; dims[3] = ncol;
    strides[0] = m * 8; strides[1] = m * m * 8; strides[2] = ld * 8;
    box[0] = ubox ? QU3X : QB3X; box[1] = ubox ? QU3Y : QV3Y; box[2] = ubox ? QU3Z : QV3Z; box[3] = 1;
  } else {
    rank = 3;
    dims[0] = m; dims[1] = nz + 2 * G; dims[2] = ncol;
    strides[0] = m * 8; strides[1] = ld * 8;
    box[0] = ubox ? QU2X : QB2X; box[1] = ubox ? QU2Y : QV2Y; box[2] = 1;
  }
  CUresult r = g_encode(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<double*>(base), dims, strides, box,
                        es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

struct StencilMaps {
  CUtensorMap WU, WV, XU, FV, VU;
  MapKey key[6];
};

static size_t tma_smem(int dim, int KM, int NST) {
  if (dim == 3) return 128 + sizeof(double) * ((size_t)NST * (QU3 + (KM - 1) * QB3) + QV3P);
  return 128 + sizeof(double) * ((size_t)NST * (QU2 + (KM - 1) * QB2P) + QV2P);
}

static int tma_env(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}

static int tma_nst(int dim, int KM) {
  const int want = tma_env("SKS_TMA_NST", 2);
  const size_t lim = 200 * 1024;
  if (want == 1 && tma_smem(dim, KM, 1) <= lim) return 1;
  if (tma_smem(dim, KM, 2) <= lim) return 2;
  if (tma_smem(dim, KM, 1) <= lim) return 1;
  return 0;
}

bool stencil_tma_supported(int dim, int64_t m, int k) {
  if (m % 2) return false;  // TMA global strides must be multiples of 16 bytes
  return tma_nst(dim, step_km(k)) > 0 && get_encode();
}

template <int KM, int NST>
static cudaError_t launch_t(const StepArgs& a, const TmaCols& tc, const CUtensorMap& mu, const CUtensorMap& mv,
                            int grid, cudaStream_t st) {
  const size_t smem = tma_smem(a.dim, KM, NST);
  if (a.dim == 3) {
    if (cudaError_t e = set_smem_attr(step3d_tma_kernel<KM, NST>, smem)) return e;
    return launch_pdl(step3d_tma_kernel<KM, NST>, grid, QT, smem, st, a, tc, mu, mv);
  } else {
    if (cudaError_t e = set_smem_attr(step2d_tma_kernel<KM, NST>, smem)) return e;
    return launch_pdl(step2d_tma_kernel<KM, NST>, grid, QT, smem, st, a, tc, mu, mv);
  }
  return cudaGetLastError();
}

template <int KM>
static cudaError_t launch_km(const StepArgs& a, const TmaCols& tc, const CUtensorMap& mu, const CUtensorMap& mv,
                             int grid, cudaStream_t st) {
  const int nst = tma_nst(a.dim, KM);
  if (nst == 2) return launch_t<KM, 2>(a, tc, mu, mv, grid, st);
  if (nst == 1) return launch_t<KM, 1>(a, tc, mu, mv, grid, st);
  return cudaErrorInvalidConfiguration;
}

// tiling + persistent grid for the TMA kernels
void stencil_tma_tiling(int dim, int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid) {
  if (dim == 3) {
    a->tiles_x = (int)((m + Q3X - 1) / Q3X);
    a->tiles_y = (int)((m + Q3Y - 1) / Q3Y);
    const int64_t tz = (nz + Q3Z - 1) / Q3Z;
    a->ntiles = (int64_t)a->tiles_x * a->tiles_y * tz;
  } else {
    a->tiles_x = (int)((m + Q2X - 1) / Q2X);
    a->tiles_y = (int)((nz + Q2Y - 1) / Q2Y);
    a->ntiles = (int64_t)a->tiles_x * a->tiles_y;
  }
  a->zchunk = 0;
  *grid = (int)std::max<int64_t>(1, std::min<int64_t>(a->ntiles, (int64_t)num_sms * tma_env("SKS_TMA_CPS", 1)));
}

// mode 0: U = column j-1, V_l = columns lo+l of W; mode 1: U = x, V0 = f; mode 2: U = v0.
cudaError_t launch_step_stencil_tma(const StepArgs& a, const double* W, int64_t ncol, const double* xb,
                                    const double* fb, const double* vb, int grid, cudaStream_t st, void** cache) {
  StencilMaps* mp = reinterpret_cast<StencilMaps*>(*cache);
  if (!mp) {
    mp = new StencilMaps();
    *cache = mp;
  }
  auto upd = [&](CUtensorMap* mpp, int slot, const double* base, int64_t nc, bool ub) -> bool {
    // re-encode when the base pointer or any field of the geometry changes (exact comparison)
    MapKey key;
    key.base = base;
    key.ld = a.ld;
    key.nz = a.nz;
    key.m = a.m;
    key.ncol = nc;
    key.G = a.G;
    key.depth = a.dim;
    key.kind = ub ? 1 : 0;
    if (mp->key[slot] == key) return true;
    if (!encode_map(mpp, a.dim, base, a.m, a.nz, a.G, a.ld, nc, ub)) return false;
    mp->key[slot] = key;
    return true;
  };
  TmaCols tc;
  memset(&tc, 0, sizeof(tc));
  tc.nv = (a.mode == 0) ? std::min(a.j, a.k) - 1 : (a.mode == 1 ? 1 : 0);  // = StepCoef::nv
  const CUtensorMap* mu;
  const CUtensorMap* mv;
  if (a.mode == 0) {
    if (!upd(&mp->WU, 0, W, ncol, true) || !upd(&mp->WV, 1, W, ncol, false)) return cudaErrorInvalidValue;
    mu = &mp->WU;
    mv = &mp->WV;
    const int lo = std::max(0, a.j - a.k);
    tc.ucol = a.j - 1;
    for (int l = 0; l < a.j - 1 - lo; ++l) tc.vcol[l] = lo + l;
  } else if (a.mode == 1) {
    if (!upd(&mp->XU, 2, xb, 1, true) || !upd(&mp->FV, 3, fb, 1, false)) return cudaErrorInvalidValue;
    mu = &mp->XU;
    mv = &mp->FV;
  } else {
    if (!upd(&mp->VU, 4, vb, 1, true)) return cudaErrorInvalidValue;
    if (!upd(&mp->WV, 1, W, ncol, false)) return cudaErrorInvalidValue;
    mu = &mp->VU;
    mv = &mp->WV;  // unused (nv = 0)
  }
  switch (step_km(a.k)) {
    case 2: return launch_km<2>(a, tc, *mu, *mv, grid, st);
    case 4: return launch_km<4>(a, tc, *mu, *mv, grid, st);
    default: return launch_km<8>(a, tc, *mu, *mv, grid, st);
  }
}

void stencil_tma_free(void* cache) { delete reinterpret_cast<StencilMaps*>(cache); }

}  // namespace sks
