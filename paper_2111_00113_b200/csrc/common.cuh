// common.cuh -- shared device/host helpers of libsks (product side; shares nothing with oracle/).
#pragma once
#include <cuda_runtime.h>
#include <cstdlib>
#include <stdint.h>
#include <math.h>

#define SKS_KMAX 8          // max partial-orthogonalisation window k
#define SKS_NP (SKS_KMAX + 3)  // partials per step kernel: ||w||^2, <w,Aw>, ||Aw||^2, k-1 window dots
#define SKS_SMAX 2048       // max sketch rows
#define SKS_JB 32           // max columns per sketch batch (one warp lane per column)
#define SKS_ZETA_MAX 16

// ---------------------------------------------------------------------------------
// Counter-based hash of the sparse sign map S (reading O5 in DESIGN.md).
// Integer-only, so the device table is bit-identical to the spec.
//   fmix64 = splitmix64 finaliser; key(seed,c) = fmix64(fmix64(seed ^ DOMAIN) + G*(c+1))
//   word(r,t) = fmix64(key + G*(16 r + t)); draws u_t = 32-bit halves of words 0..7;
//   sign word = word(r, 8); Floyd: J = s-zeta+t, v = (u_t*(J+1))>>32, q_t = v or J.
// ---------------------------------------------------------------------------------
#define SKS_GAMMA 0x9E3779B97F4A7C15ULL
#define SKS_DOMAIN 0x736B732D534B4554ULL

__host__ __device__ __forceinline__ uint64_t sks_fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

__host__ __device__ __forceinline__ uint64_t sks_key(uint64_t seed, uint32_t cycle) {
  return sks_fmix64(sks_fmix64(seed ^ SKS_DOMAIN) + SKS_GAMMA * (uint64_t)(cycle + 1u));
}

// (row, sign) entries of column `r` of S: q[t] in [0,s), neg bit t of *negmask.
template <int ZETA>
__device__ __forceinline__ void sks_column(uint64_t key, uint64_t r, int s, int* q, uint32_t* negmask) {
  const uint64_t base = key + SKS_GAMMA * (16ull * r);
#pragma unroll
  for (int t = 0; t < ZETA; ++t) {
    uint64_t w = sks_fmix64(base + SKS_GAMMA * (uint64_t)(t >> 1));
    uint32_t u = (t & 1) ? (uint32_t)(w >> 32) : (uint32_t)(w & 0xffffffffu);
    const uint32_t J = (uint32_t)(s - ZETA + t);
    uint32_t v = (uint32_t)(((uint64_t)u * (uint64_t)(J + 1u)) >> 32);
    bool taken = false;
#pragma unroll
    for (int i = 0; i < t; ++i) taken |= (q[i] == (int)v);
    q[t] = taken ? (int)J : (int)v;
  }
  *negmask = (uint32_t)(sks_fmix64(base + SKS_GAMMA * 8ull) & ((1ull << ZETA) - 1ull));
}

// runtime-zeta variant (<= 16), used by the table entry point and generic sketch path
__device__ __forceinline__ void sks_column_rt(uint64_t key, uint64_t r, int s, int zeta, int* q,
                                              uint32_t* negmask) {
  const uint64_t base = key + SKS_GAMMA * (16ull * r);
  uint64_t w = 0;
  for (int t = 0; t < zeta; ++t) {
    if ((t & 1) == 0) w = sks_fmix64(base + SKS_GAMMA * (uint64_t)(t >> 1));
    uint32_t u = (t & 1) ? (uint32_t)(w >> 32) : (uint32_t)(w & 0xffffffffu);
    const uint32_t J = (uint32_t)(s - zeta + t);
    uint32_t v = (uint32_t)(((uint64_t)u * (uint64_t)(J + 1u)) >> 32);
    bool taken = false;
    for (int i = 0; i < t; ++i) taken |= (q[i] == (int)v);
    q[t] = taken ? (int)J : (int)v;
  }
  *negmask = (uint32_t)(sks_fmix64(base + SKS_GAMMA * 8ull) & ((1ull << zeta) - 1ull));
}

// ---------------------------------------------------------------------------------
// reductions (deterministic: fixed shuffle tree, fixed smem tree)
// ---------------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// block-wide sum of NV values per thread; result valid in thread 0 (out[]); smem >= NV*32 doubles
template <int NV>
__device__ __forceinline__ void block_sum_n(double (&v)[NV], double* smem, double* out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = warp_sum(v[i]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) smem[i * 32 + wid] = v[i];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      double t = lane < nw ? smem[i * 32 + lane] : 0.0;
      t = warp_sum(t);
      if (lane == 0) out[i] = t;
    }
  }
  __syncthreads();
}

__device__ __forceinline__ double block_sum(double v, double* smem) {
  double a[1] = {v};
  double o[1];
  __shared__ double res;
  block_sum_n<1>(a, smem, o);
  if (threadIdx.x == 0) res = o[0];
  __syncthreads();
  double r = res;
  __syncthreads();
  return r;
}

// ---------------------------------------------------------------------------------
// device-side control block of one solve (written by kernels, read by kernels/host)
// ---------------------------------------------------------------------------------
struct CtrlBlock {
  int stop_col;       // first column that must NOT be used (breakdown), INT_MAX if none
  int breakdown;      // 1 if breakdown detected
  int exit_cols;      // early exit: number of columns of the chosen solution (0 = not yet)
  int qr_cols;        // columns appended to the sketched QR so far
  int rank_def;       // sketched QR hit a (numerically) zero column
  int pad[3];
  double rnorm;       // ||r|| of the current cycle's residual (written by step kernel j=1)
  double fnorm;       // ||f||
  double thr;         // early-exit threshold on r_est (absolute)
  double cond;        // kappa estimate of T
  double r_est_last;  // r_est at exit / last appended column
  double pad2[3];
};

namespace sks {
// ---- programmatic dependent launch (PDL) for the back-to-back basis-step kernels: a step grid may be
// scheduled while the previous kernel on the stream drains; it runs its set-up (barrier init, tensor
// map prefetch), then waits for that kernel's completion before reading any of its outputs.
__device__ __forceinline__ void pdl_wait_and_release() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
}
inline bool pdl_enabled() {  // SKS_NO_PDL=1 turns it off (A/B measurements)
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SKS_NO_PDL");
    on = (e && e[0] == '1') ? 0 : 1;
  }
  return on == 1;
}
// cudaFuncAttributeMaxDynamicSharedMemorySize is a per-device function attribute: set_smem_attr
// remembers, per (kernel, current device), the largest size already set (api.cu; thread-safe).
cudaError_t set_smem_attr_raw(const void* fn, size_t smem);
template <typename K>
inline cudaError_t set_smem_attr(K* kern, size_t smem) {
  return set_smem_attr_raw(reinterpret_cast<const void*>(kern), smem);
}

// identity of an encoded CUtensorMap: every field that enters the encoding, compared exactly
struct MapKey {
  const void* base = nullptr;
  int64_t ld = -1, nz = -1, m = -1, ncol = -1;
  int G = -1, depth = -1, kind = -1;
  bool operator==(const MapKey& o) const {
    return base == o.base && ld == o.ld && nz == o.nz && m == o.m && ncol == o.ncol && G == o.G &&
           depth == o.depth && kind == o.kind;
  }
};

template <typename K, typename... Args>
inline cudaError_t launch_pdl(K kern, int grid, int block, size_t smem, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}
}  // namespace sks
