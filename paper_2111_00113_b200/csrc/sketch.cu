// sketch.cu -- S M for a batch of up to 32 columns M (sparse sign map).
//
// Formulation: S is regenerated from the counter hash
// (common.cuh) and never stored.  Each CTA owns a contiguous range of rows and walks it
// in tiles of R rows.  Per tile:
//   1. stage M[tile rows, 0..J) in shared memory as Mt[r][c] (row-major, 32 columns),
//   2. hash the tile's rows -> zeta (q, sign) entries per row, counting-sort them by q
//      (deterministic: buckets re-sorted by row),
//   3. GATHER: warp w / lane c owns sketch rows q = w + 16 i and column c and keeps
//      acc[i] = sum over its bucket entries of +-Mt[r][c] in REGISTERS.
// The gather needs no atomics and reads shared memory conflict-free (a warp reads one
// 256-byte row of Mt per entry).  Per-CTA partial sketches are summed in a fixed order
// by a second kernel, so the result is bitwise reproducible.
#include "common.cuh"
#include "internal.h"

namespace sks {

constexpr int SK_R = 512;       // rows per tile
constexpr int SK_THREADS = 512; // 16 warps; one row hashed per thread
constexpr int SK_WARPS = SK_THREADS / 32;

struct SketchArgs {
  const double* M;   // column c at M + c*ldm
  int64_t ldm;
  int64_t nrows;     // local rows
  int64_t row_begin; // global index of local row 0
  int J;             // columns in this batch (<= 32)
  int s, zeta;
  int q_base;        // first sketch row handled by this pass
  uint64_t key;
  double scale;      // 1/sqrt(zeta)
  double* part;      // [grid][J][s] partial sketches (this pass writes q in [q_base, q_base+16*QPW))
  int64_t tiles;     // ceil(nrows / SK_R)
  int vec_ok;        // 16-byte vector loads allowed
};

// Shared-memory layout (bytes):  Mt[SK_R][32] doubles | cnt[s+1] | cur[s] | tab[SK_R*zeta] u16 | ent[SK_R*zeta] u32
template <int QPW, int ZETA>
__global__ void __launch_bounds__(SK_THREADS, 1) sketch_batch_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* Mt = reinterpret_cast<double*>(smraw);                    // [SK_R][32]
  int* cnt = reinterpret_cast<int*>(Mt + SK_R * 32);                // [s+1] bucket starts
  int* cur = cnt + (a.s + 1);                                       // [s]
  uint16_t* tab = reinterpret_cast<uint16_t*>(cur + a.s);            // [SK_R*zeta] (q | neg<<15) per (row,t)
  uint32_t* ent = reinterpret_cast<uint32_t*>(tab + ((SK_R * SKS_ZETA_MAX + 1) & ~1));  // sorted: byte offset | neg<<31
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s = a.s;
  const int zeta = ZETA > 0 ? ZETA : a.zeta;
  const unsigned char* mtl = reinterpret_cast<const unsigned char*>(Mt) + lane * 8;  // this lane's column
  // this warp owns the contiguous sketch-row block [qlo, qlo + QPW)
  const int qlo = a.q_base + wid * QPW;
  double acc[QPW];
#pragma unroll
  for (int i = 0; i < QPW; ++i) acc[i] = 0.0;

  const int64_t t_lo = (a.tiles * blockIdx.x) / gridDim.x;
  const int64_t t_hi = (a.tiles * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t tile = t_lo; tile < t_hi; ++tile) {
    const int64_t r0 = tile * SK_R;
    const int nr = (int)((a.nrows - r0) < (int64_t)SK_R ? (a.nrows - r0) : (int64_t)SK_R);
    // ---- 1. stage Mt (two halves: 4 x 32-byte loads in flight per thread each)
    if (a.vec_ok) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        constexpr int NIT = (SK_R / 4) * 32 / SK_THREADS / 2;  // 4
        double2 va[NIT], vb[NIT];
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
          const int idx = tid + (half * NIT + u) * SK_THREADS;
          const int r = (idx >> 5) * 4, c = idx & 31;
          va[u] = make_double2(0.0, 0.0);
          vb[u] = make_double2(0.0, 0.0);
          if (c < a.J) {
            const double* src = a.M + (int64_t)c * a.ldm + r0 + r;
            if (r + 3 < nr) {
              va[u] = __ldg(reinterpret_cast<const double2*>(src));
              vb[u] = __ldg(reinterpret_cast<const double2*>(src + 2));
            } else {
              if (r + 0 < nr) va[u].x = src[0];
              if (r + 1 < nr) va[u].y = src[1];
              if (r + 2 < nr) vb[u].x = src[2];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
          const int idx = tid + (half * NIT + u) * SK_THREADS;
          const int r = (idx >> 5) * 4, c = idx & 31;
          Mt[(r + 0) * 32 + c] = va[u].x;
          Mt[(r + 1) * 32 + c] = va[u].y;
          Mt[(r + 2) * 32 + c] = vb[u].x;
          Mt[(r + 3) * 32 + c] = vb[u].y;
        }
      }
    } else {
      for (int idx = tid; idx < SK_R * 32; idx += SK_THREADS) {
        const int r = idx >> 5, c = idx & 31;
        double v = 0.0;
        if (c < a.J && r < nr) v = a.M[(int64_t)c * a.ldm + r0 + r];
        Mt[idx] = v;
      }
    }
    // ---- 2. hash (one row per thread) + counting sort by sketch row
    for (int q = tid; q <= s; q += SK_THREADS) cnt[q] = 0;
    __syncthreads();
    if (tid < nr) {
      int qq[ZETA > 0 ? ZETA : SKS_ZETA_MAX];
      uint32_t neg;
      if (ZETA > 0)
        sks_column<(ZETA > 0 ? ZETA : 1)>(a.key, (uint64_t)(a.row_begin + r0 + tid), s, qq, &neg);
      else
        sks_column_rt(a.key, (uint64_t)(a.row_begin + r0 + tid), s, zeta, qq, &neg);
#pragma unroll
      for (int t = 0; t < (ZETA > 0 ? ZETA : SKS_ZETA_MAX); ++t) {
        if (t < zeta) {
          atomicAdd(&cnt[qq[t]], 1);
          tab[tid * zeta + t] = (uint16_t)(qq[t] | (((neg >> t) & 1u) << 15));
        }
      }
    }
    __syncthreads();
    if (wid == 0) {  // exclusive scan of cnt[0..s) by one warp
      int carry = 0;
      for (int base = 0; base < s; base += 32) {
        const int q = base + lane;
        const int v = q < s ? cnt[q] : 0;
        int incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += t;
        }
        if (q < s) {
          cnt[q] = carry + incl - v;
          cur[q] = carry + incl - v;
        }
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) cnt[s] = carry;
    }
    __syncthreads();
    if (tid < nr) {
      for (int t = 0; t < zeta; ++t) {
        const uint16_t e = tab[tid * zeta + t];
        const int q = e & 0x7fff;
        const int pos = atomicAdd(&cur[q], 1);
        ent[pos] = (uint32_t)(tid * 256) | ((uint32_t)(e & 0x8000) << 16);  // byte offset of row tid | sign
      }
    }
    __syncthreads();
    for (int q = tid; q < s; q += SK_THREADS) {  // deterministic order inside a bucket (by row)
      const int b = cnt[q], e = cnt[q + 1];
      for (int i = b + 1; i < e; ++i) {
        const uint32_t key = ent[i];
        int j = i - 1;
        while (j >= b && (ent[j] & 0x7fffffffu) > (key & 0x7fffffffu)) {
          ent[j + 1] = ent[j];
          --j;
        }
        ent[j + 1] = key;
      }
    }
    __syncthreads();
    // ---- 3. gather: walk this warp's contiguous entry segment bucket by bucket
    {
      int p = cnt[qlo < s ? qlo : s];
#pragma unroll
      for (int i = 0; i < QPW; ++i) {
        const int q = qlo + i;
        const int e = (q < s) ? cnt[q + 1] : p;
        double t0 = 0.0, t1 = 0.0;
        for (; p + 1 < e; p += 2) {
          const uint32_t e0 = ent[p], e1 = ent[p + 1];
          const double x0 = *reinterpret_cast<const double*>(mtl + (e0 & 0x7fffffffu));
          const double x1 = *reinterpret_cast<const double*>(mtl + (e1 & 0x7fffffffu));
          t0 += __hiloint2double(__double2hiint(x0) ^ (int)(e0 & 0x80000000u), __double2loint(x0));
          t1 += __hiloint2double(__double2hiint(x1) ^ (int)(e1 & 0x80000000u), __double2loint(x1));
        }
        if (p < e) {
          const uint32_t e0 = ent[p];
          const double x0 = *reinterpret_cast<const double*>(mtl + (e0 & 0x7fffffffu));
          t0 += __hiloint2double(__double2hiint(x0) ^ (int)(e0 & 0x80000000u), __double2loint(x0));
          ++p;
        }
        acc[i] += t0 + t1;
      }
    }
    __syncthreads();
  }
  // ---- partial sketch of this CTA
  if (lane < a.J) {
#pragma unroll
    for (int i = 0; i < QPW; ++i) {
      const int q = qlo + i;
      if (q < s) a.part[((int64_t)blockIdx.x * a.J + lane) * s + q] = acc[i] * a.scale;
    }
  }
}

// ------------------------------------------------------------------------------
// v3 (s <= 768): deterministic placement without atomics or sorting.  Entries are keyed
// k = 2q + sign; each warp ranks its own entries per key with __match_any_sync (order
// (t, lane)), per-key warp offsets come from a prefix over the 16 warps, so a bucket
// holds [positive entries | negative entries] in (warp, t, lane) order -- bitwise
// reproducible -- and the gather needs no per-entry sign handling.
// ------------------------------------------------------------------------------
constexpr int S3_NKMAX = 1536;  // 2 s

static __device__ __forceinline__ double mt_at(const unsigned char* mtl, uint32_t off) {
  return *reinterpret_cast<const double*>(mtl + off);
}

template <int QPW, int ZETA>
__global__ void __launch_bounds__(SK_THREADS, 1) sketch_v3_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double* Mt = reinterpret_cast<double*>(smraw);                      // [SK_R][32]
  __shared__ int wsum[SK_WARPS];
  __shared__ double sstage[SK_WARPS * 8 * 32];                        // per-warp bucket sums (8 q x 32 cols)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int s = a.s, NK = 2 * s, NKP = (NK + 7) & ~7;
  constexpr int Z = ZETA > 0 ? ZETA : SKS_ZETA_MAX;
  const int zeta = ZETA > 0 ? ZETA : a.zeta;
  // dynamic layout sized by (s, zeta): see sketch_v3_smem()
  uint32_t* ent = reinterpret_cast<uint32_t*>(Mt + SK_R * 32);         // [SK_R * zeta] row byte offsets
  int* kst = reinterpret_cast<int*>(ent + SK_R * zeta);                // [NKP + 8] key starts
  uint16_t* wc = reinterpret_cast<uint16_t*>(kst + NKP + 8);           // [16][NKP] per-warp key counts/offsets
  const unsigned char* mtl = reinterpret_cast<const unsigned char*>(Mt) + lane * 8;
  const int qlo = a.q_base + wid * QPW;
  const uint32_t ltmask = (1u << lane) - 1u;
  double acc[QPW];
#pragma unroll
  for (int i = 0; i < QPW; ++i) acc[i] = 0.0;

  const int64_t t_lo = (a.tiles * blockIdx.x) / gridDim.x;
  const int64_t t_hi = (a.tiles * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t tile = t_lo; tile < t_hi; ++tile) {
    const int64_t r0 = tile * SK_R;
    const int nr = (int)((a.nrows - r0) < (int64_t)SK_R ? (a.nrows - r0) : (int64_t)SK_R);
    // ---- 1. stage Mt[r][c] (row-major, 32 columns)
    if (a.vec_ok) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        constexpr int NIT = (SK_R / 4) * 32 / SK_THREADS / 2;
        double2 va[NIT], vb[NIT];
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
          const int idx = tid + (half * NIT + u) * SK_THREADS;
          const int r = (idx >> 5) * 4, c = idx & 31;
          va[u] = make_double2(0.0, 0.0);
          vb[u] = make_double2(0.0, 0.0);
          if (c < a.J) {
            const double* src = a.M + (int64_t)c * a.ldm + r0 + r;
            if (r + 3 < nr) {
              va[u] = __ldg(reinterpret_cast<const double2*>(src));
              vb[u] = __ldg(reinterpret_cast<const double2*>(src + 2));
            } else {
              if (r + 0 < nr) va[u].x = src[0];
              if (r + 1 < nr) va[u].y = src[1];
              if (r + 2 < nr) vb[u].x = src[2];
            }
          }
        }
#pragma unroll
        for (int u = 0; u < NIT; ++u) {
          const int idx = tid + (half * NIT + u) * SK_THREADS;
          const int r = (idx >> 5) * 4, c = idx & 31;
          Mt[(r + 0) * 32 + c] = va[u].x;
          Mt[(r + 1) * 32 + c] = va[u].y;
          Mt[(r + 2) * 32 + c] = vb[u].x;
          Mt[(r + 3) * 32 + c] = vb[u].y;
        }
      }
    } else {
      for (int idx = tid; idx < SK_R * 32; idx += SK_THREADS) {
        const int r = idx >> 5, c = idx & 31;
        double v = 0.0;
        if (c < a.J && r < nr) v = a.M[(int64_t)c * a.ldm + r0 + r];
        Mt[idx] = v;
      }
    }
    for (int i = tid; i < SK_WARPS * NKP / 8; i += SK_THREADS) reinterpret_cast<uint4*>(wc)[i] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    // ---- 2. hash this thread's row; warp-local ranks per key
    const bool valid = tid < nr;
    int key[Z];
    {
      int qq[Z];
      uint32_t neg = 0;
      if (valid) {
        if (ZETA > 0)
          sks_column<(ZETA > 0 ? ZETA : 1)>(a.key, (uint64_t)(a.row_begin + r0 + tid), s, qq, &neg);
        else
          sks_column_rt(a.key, (uint64_t)(a.row_begin + r0 + tid), s, zeta, qq, &neg);
      }
#pragma unroll
      for (int t = 0; t < Z; ++t) key[t] = (valid && t < zeta) ? 2 * qq[t] + (int)((neg >> t) & 1u) : -1 - lane;
    }
    uint16_t pos[Z];
#pragma unroll
    for (int t = 0; t < Z; ++t) {
      if (t < zeta) {
        const uint32_t mm = __match_any_sync(0xffffffffu, key[t]);
        const int rank = __popc(mm & ltmask);
        int base = 0;
        if (key[t] >= 0) base = wc[wid * NKP + key[t]];
        pos[t] = (uint16_t)(base + rank);
        __syncwarp();
        if (key[t] >= 0 && lane == __ffs(mm) - 1) wc[wid * NKP + key[t]] = (uint16_t)(base + __popc(mm));
        __syncwarp();
      }
    }
    __syncthreads();
    // ---- 3. per-key prefix over warps, then exclusive scan over keys
    for (int k = tid; k < NK; k += SK_THREADS) {
      int run = 0;
#pragma unroll
      for (int w = 0; w < SK_WARPS; ++w) {
        const int c = wc[w * NKP + k];
        wc[w * NKP + k] = (uint16_t)run;
        run += c;
      }
      kst[k] = run;
    }
    __syncthreads();
    {
      constexpr int CH = (S3_NKMAX + SK_THREADS - 1) / SK_THREADS;  // 3 keys per thread
      int v[CH];
      int loc = 0;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int k = tid * CH + i;
        v[i] = (k < NK) ? kst[k] : 0;
        loc += v[i];
      }
      int incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum[wid] = incl;
      __syncthreads();
      int wbase = 0;
      for (int w = 0; w < wid; ++w) wbase += wsum[w];
      int ex = wbase + incl - loc;
#pragma unroll
      for (int i = 0; i < CH; ++i) {
        const int k = tid * CH + i;
        if (k < NK) kst[k] = ex;
        ex += v[i];
      }
      if (tid == SK_THREADS - 1) kst[NK] = ex;
    }
    __syncthreads();
    for (int k = tid; k < NK; k += SK_THREADS) {
      const int b = kst[k];
#pragma unroll
      for (int w = 0; w < SK_WARPS; ++w) wc[w * NKP + k] = (uint16_t)(wc[w * NKP + k] + b);
    }
    __syncthreads();
    // ---- 4. place entries (row byte offsets)
    if (valid) {
#pragma unroll
      for (int t = 0; t < Z; ++t)
        if (t < zeta) ent[wc[wid * NKP + key[t]] + pos[t]] = (uint32_t)(tid * 256);
    }
    __syncthreads();
    // ---- 5. gather: bucket q = [positives | negatives].  The q loop is NOT unrolled (compact
    //         code); each bucket sum goes to a per-warp shared staging row and is folded into
    //         the register accumulators 8 at a time by a small unrolled loop.
    {
      double* stg = sstage + wid * 8 * 32 + lane;
      int p = kst[2 * (qlo < s ? qlo : s)];
#pragma unroll
      for (int ch = 0; ch < QPW / 8; ++ch) {
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
          const int q = qlo + ch * 8 + k;
          double tsum = 0.0;
          if (q < s) {
            const int ep = kst[2 * q + 1], en = kst[2 * q + 2];
            double a0 = 0.0, a1 = 0.0, b0 = 0.0, b1 = 0.0;
#pragma unroll 1
            for (; p + 1 < ep; p += 2) {
              a0 += mt_at(mtl, ent[p]);
              a1 += mt_at(mtl, ent[p + 1]);
            }
            if (p < ep) a0 += mt_at(mtl, ent[p++]);
#pragma unroll 1
            for (; p + 1 < en; p += 2) {
              b0 += mt_at(mtl, ent[p]);
              b1 += mt_at(mtl, ent[p + 1]);
            }
            if (p < en) b0 += mt_at(mtl, ent[p++]);
            tsum = (a0 + a1) - (b0 + b1);
          }
          stg[k * 32] = tsum;
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < 8; ++k) acc[ch * 8 + k] += stg[k * 32];
        __syncwarp();
      }
    }
    __syncthreads();
  }
  if (lane < a.J) {
#pragma unroll
    for (int i = 0; i < QPW; ++i) {
      const int q = qlo + i;
      if (q < s) a.part[((int64_t)blockIdx.x * a.J + lane) * s + q] = acc[i] * a.scale;
    }
  }
}

// out[c*ldo + q] (+)= sum_b part[b][c][q]  (fixed order over b)
__global__ void sketch_reduce_kernel(const double* __restrict__ part, int grid, int J, int s,
                                     double* __restrict__ out, int64_t ldo, int accumulate) {
  const int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (idx >= (int64_t)J * s) return;
  const int c = (int)(idx / s), q = (int)(idx % s);
  double t = 0.0;
  for (int b = 0; b < grid; ++b) t += part[((int64_t)b * J + c) * s + q];
  if (accumulate) out[(int64_t)c * ldo + q] += t;
  else out[(int64_t)c * ldo + q] = t;
}

__global__ void sketch_table_kernel(int64_t row_begin, int64_t count, int s, int zeta, uint64_t key,
                                    int32_t* __restrict__ q, int8_t* __restrict__ sign) {
  const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (r >= count) return;
  int qq[SKS_ZETA_MAX];
  uint32_t neg;
  sks_column_rt(key, (uint64_t)(row_begin + r), s, zeta, qq, &neg);
  for (int t = 0; t < zeta; ++t) {
    q[r * zeta + t] = qq[t];
    sign[r * zeta + t] = ((neg >> t) & 1u) ? (int8_t)-1 : (int8_t)1;
  }
}

// ------------------------------------------------------------------------------
static size_t sketch_smem(int s) {
  return sizeof(double) * SK_R * 32 + sizeof(int) * (2 * s + 1) + sizeof(uint16_t) * ((SK_R * SKS_ZETA_MAX + 1) & ~1) +
         sizeof(uint32_t) * SK_R * SKS_ZETA_MAX + 32;
}

template <int QPW, int ZETA>
static cudaError_t launch_sk(const SketchArgs& a, int grid, cudaStream_t st) {
  const size_t smem = sketch_smem(a.s);
  static size_t set = 0;
  if (set < smem) {
    cudaError_t e = cudaFuncSetAttribute(sketch_batch_kernel<QPW, ZETA>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    set = smem;
  }
  sketch_batch_kernel<QPW, ZETA><<<grid, SK_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

// dynamic shared memory of sketch_v3_kernel for (s, zeta); its static part is sstage+wsum
static size_t sketch_v3_smem(int s, int zeta) {
  const size_t nkp = (size_t)((2 * s + 7) & ~7);
  return sizeof(double) * SK_R * 32 + sizeof(uint32_t) * SK_R * zeta + sizeof(int) * (nkp + 8) +
         sizeof(uint16_t) * SK_WARPS * nkp + 64;
}
constexpr size_t SK3_STATIC = sizeof(double) * SK_WARPS * 8 * 32 + sizeof(int) * SK_WARPS + 256;

static bool sketch_v3_fits(int s, int zeta) {
  static int optin = 0;
  if (!optin) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
      cudaGetLastError();
      optin = 232448;
    }
  }
  return 2 * s <= S3_NKMAX && sketch_v3_smem(s, zeta) + SK3_STATIC <= (size_t)optin;
}

template <int QPW, int ZETA>
static cudaError_t launch_v3(const SketchArgs& a, int grid, cudaStream_t st) {
  const size_t smem = sketch_v3_smem(a.s, a.zeta);
  static size_t set = 0;
  if (set < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(sketch_v3_kernel<QPW, ZETA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    set = smem;
  }
  sketch_v3_kernel<QPW, ZETA><<<grid, SK_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

template <int ZETA>
static cudaError_t launch_v3_z(const SketchArgs& a, int grid, cudaStream_t st) {
  const int span = a.s;
  if (span <= 8 * SK_WARPS) return launch_v3<8, ZETA>(a, grid, st);
  if (span <= 16 * SK_WARPS) return launch_v3<16, ZETA>(a, grid, st);
  if (span <= 24 * SK_WARPS) return launch_v3<24, ZETA>(a, grid, st);
  if (span <= 32 * SK_WARPS) return launch_v3<32, ZETA>(a, grid, st);
  if (span <= 40 * SK_WARPS) return launch_v3<40, ZETA>(a, grid, st);
  return launch_v3<48, ZETA>(a, grid, st);
}

template <int ZETA>
static cudaError_t launch_sk_z(const SketchArgs& a, int qspan, int grid, cudaStream_t st) {
  if (qspan <= 8 * SK_WARPS) return launch_sk<8, ZETA>(a, grid, st);
  if (qspan <= 16 * SK_WARPS) return launch_sk<16, ZETA>(a, grid, st);
  if (qspan <= 24 * SK_WARPS) return launch_sk<24, ZETA>(a, grid, st);
  if (qspan <= 32 * SK_WARPS) return launch_sk<32, ZETA>(a, grid, st);
  return launch_sk<40, ZETA>(a, grid, st);
}

int sketch_grid(int num_sms, int64_t nrows) {
  int64_t tiles = (nrows + SK_R - 1) / SK_R;
  return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms));
}

size_t sketch_part_doubles(int grid, int J, int s) { return (size_t)grid * J * s; }

// SM[:, 0..J) (column-major, ld = ldo) = S_key M[:, 0..J) for rows [row_begin, row_begin+nrows)
cudaError_t launch_sketch(const double* M, int64_t ldm, int64_t nrows, int64_t row_begin, int J, int s,
                          int zeta, uint64_t key, double* part, int grid, double* out, int64_t ldo,
                          int accumulate, cudaStream_t st, int64_t* launches) {
  if (J < 1 || J > SKS_JB) return cudaErrorInvalidValue;
  SketchArgs a;
  a.M = M;
  a.ldm = ldm;
  a.nrows = nrows;
  a.row_begin = row_begin;
  a.J = J;
  a.s = s;
  a.zeta = zeta;
  a.key = key;
  a.scale = 1.0 / sqrt((double)zeta);
  a.part = part;
  a.tiles = (nrows + SK_R - 1) / SK_R;
  a.vec_ok = ((((uintptr_t)M) & 15) == 0) && (ldm % 2 == 0);
  if (sketch_v3_fits(s, zeta)) {
    a.q_base = 0;
    cudaError_t e = (zeta == 8) ? launch_v3_z<8>(a, grid, st) : launch_v3_z<0>(a, grid, st);
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
    const int64_t tot = (int64_t)J * s;
    sketch_reduce_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(part, grid, J, s, out, ldo, accumulate);
    if (launches) ++*launches;
    return cudaGetLastError();
  }
  const int span_max = 40 * SK_WARPS;
  for (int qb = 0; qb < s; qb += span_max) {
    a.q_base = qb;
    const int span = std::min(span_max, s - qb);
    cudaError_t e = (zeta == 8) ? launch_sk_z<8>(a, span, grid, st) : launch_sk_z<0>(a, span, grid, st);
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
  }
  const int64_t tot = (int64_t)J * s;
  sketch_reduce_kernel<<<(int)((tot + 255) / 256), 256, 0, st>>>(part, grid, J, s, out, ldo, accumulate);
  if (launches) ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_sketch_table(int64_t row_begin, int64_t count, int s, int zeta, uint64_t key, int32_t* q,
                                int8_t* sign, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  sketch_table_kernel<<<(int)((count + 255) / 256), 256, 0, st>>>(row_begin, count, s, zeta, key, q, sign);
  return cudaGetLastError();
}

}  // namespace sks
