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
// v4 (s <= 768): swizzled row-major staging by cp.async, deterministic counting sort by
// sketch row q without atomics, and a register gather at 32 warps per SM.
//
//  * Mt[r][c] (R = 512 rows + one zero row, 32 columns) lives at byte offset
//    r*256 + 8*(c ^ g(r&3)), g = {0, 8, 1, 9}: a 32-byte global sector (4 rows of one column)
//    lands in 4 distinct bank pairs, a staging warp (4 rows x 8 columns) and a gather warp
//    (one row, lane = column) are both conflict free, and the gather address is
//    (E ^ 8*lane) & 0x7fffffff with E = r*256 + 8*g(r&3) | sign<<31 stored per entry.
//  * Entries of one tile are bucketed by q (both signs in one bucket; the sign is an XOR
//    on the value's high word).  Placement order inside a bucket is (warp, t, lane):
//    per-warp ranks come from __match_any_sync, per-bucket warp offsets from a prefix
//    over the 16 hashing warps -- no atomics, so the result is bitwise reproducible.
//  * Every bucket is padded to an even length with an entry pointing at the zero row, so
//    the gather walks each bucket two entries at a time with no tail code.
//  * 32 warps: warp w owns sketch rows [w*QPW, (w+1)*QPW) (sums in registers, statically
//    unrolled over its buckets), lane c owns column c; 32 resident warps hide the
//    shared-memory latency of the dependent entry -> value loads.
//  * The staging of a tile is issued before its hash/sort, so the global loads overlap it.
// ------------------------------------------------------------------------------
constexpr int S4_R = 512;
constexpr int S4_QMAX = 768;
constexpr int S4_THREADS = 1024;
constexpr int S4_WARPS = S4_THREADS / 32;
constexpr int S4_HWARPS = S4_R / 32;  // warps that hash (one row per thread)

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double ld_shared_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__host__ __device__ __forceinline__ uint32_t s4_g(uint32_t r) { return r & 31u; }

// dynamic shared memory: Mt[(R+1)*32] doubles | ent[R*zeta + s + 4] u32 | kst[s + 2] int | cw[16][NQP] u16
__host__ __device__ __forceinline__ int s4_nqp(int s) { return (s + 7) & ~7; }
__host__ __device__ __forceinline__ size_t s4_ent_words(int s, int zeta) { return (size_t)S4_R * zeta + s + 4; }

template <int QPW, int ZETA>
__global__ void __launch_bounds__(S4_THREADS, 1) sketch_v4_kernel(SketchArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int Z = ZETA > 0 ? ZETA : SKS_ZETA_MAX;
  const int zeta = ZETA > 0 ? ZETA : a.zeta;
  const int s = a.s, NQP = s4_nqp(s);
  // Mt base aligned to 256 B, so an entry can carry the absolute shared address of its row
  double* Mt = reinterpret_cast<double*>(smraw + ((256u - (smem_addr(smraw) & 255u)) & 255u));
  uint32_t* ent = reinterpret_cast<uint32_t*>(Mt + (S4_R + 1) * 32);
  int* kst = reinterpret_cast<int*>(ent + s4_ent_words(s, zeta));
  uint16_t* cw = reinterpret_cast<uint16_t*>(kst + s + 2);
  __shared__ int wsum4[S4_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t lane8, amask;  // opaque to the optimiser (keeps the gather address a single LOP3)
  asm("mov.b32 %0, %1;" : "=r"(lane8) : "r"((uint32_t)lane * 8u));
  asm("mov.b32 %0, %1;" : "=r"(amask) : "r"(0x7fffffffu));
  const uint32_t mt_s = smem_addr(Mt);
  const uint32_t ltmask = (1u << lane) - 1u;
  const uint32_t PAD = mt_s + (uint32_t)S4_R * 256u;  // row R (zero); g(R) == 0
  const int qlo = wid * QPW;
  const bool hwarp = wid < S4_HWARPS;
  const uint32_t st_base = mt_s + (uint32_t)lane * 256u + 8u * ((uint32_t)(wid ^ lane) & 31u);
  uint16_t* cwm = cw + wid * NQP;
  if (tid < 32) Mt[S4_R * 32 + tid] = 0.0;

  double acc[QPW];
#pragma unroll
  for (int i = 0; i < QPW; ++i) acc[i] = 0.0;

  const int64_t t_lo = (a.tiles * blockIdx.x) / gridDim.x;
  const int64_t t_hi = (a.tiles * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t tile = t_lo; tile < t_hi; ++tile) {
    const int64_t r0 = tile * S4_R;
    const int nr = (int)((a.nrows - r0) < (int64_t)S4_R ? (a.nrows - r0) : (int64_t)S4_R);
    // ---- 1. issue the staging of Mt (async; overlaps steps 2-5).  Warp w moves column w:
    //         each instruction 32 consecutive rows (256 contiguous global bytes); the swizzle
    //         puts row r = 32 i + lane at r*256 + 8*(w ^ lane), all bank pairs distinct.
    if (wid < a.J) {
      const double* src = a.M + (int64_t)wid * a.ldm + r0 + lane;
      const uint32_t dst = st_base;
      if (nr == S4_R) {
#pragma unroll
        for (int i = 0; i < S4_R / 32; ++i) cp_async8(dst + i * 8192u, src + i * 32);
      } else {
        for (int i = 0; i < S4_R / 32; ++i)
          if (i * 32 + lane < nr) cp_async8(dst + i * 8192u, src + i * 32);
      }
    }
    // ---- 2. hash this thread's row; per-warp ranks per bucket q (hashing warps only)
    const bool valid = tid < nr;
    int kp[Z];  // bucket q (bits 0..15) | rank inside the warp's part of the bucket (bits 16..31)
    uint32_t neg = 0;
    if (hwarp) {
      for (int i = lane; i < NQP / 2; i += 32) reinterpret_cast<uint32_t*>(cwm)[i] = 0u;
      __syncwarp();
      {
        int qq[Z];
        if (valid) {
          if (ZETA > 0)
            sks_column<(ZETA > 0 ? ZETA : 1)>(a.key, (uint64_t)(a.row_begin + r0 + tid), s, qq, &neg);
          else
            sks_column_rt(a.key, (uint64_t)(a.row_begin + r0 + tid), s, zeta, qq, &neg);
        }
#pragma unroll
        for (int t = 0; t < Z; ++t) kp[t] = (valid && t < zeta) ? qq[t] : -1 - lane;
      }
#pragma unroll
      for (int t = 0; t < Z; ++t) {
        if (t < zeta) {
          const int key = kp[t];
          const uint32_t mm = __match_any_sync(0xffffffffu, key);
          const int base = (key >= 0) ? (int)cwm[key] : 0;
          kp[t] = (key & 0xffff) | ((base + __popc(mm & ltmask)) << 16);
          __syncwarp();
          if (key >= 0 && (mm & ltmask) == 0u) cwm[key] = (uint16_t)(base + __popc(mm));
          __syncwarp();
        }
      }
    }
    __syncthreads();
    // ---- 3. per-bucket prefix over the hashing warps (cw := warp offset in the bucket)
    for (int q = tid; q < s; q += S4_THREADS) {
      int run = 0;
#pragma unroll
      for (int w = 0; w < S4_HWARPS; ++w) {
        const int c = cw[w * NQP + q];
        cw[w * NQP + q] = (uint16_t)run;
        run += c;
      }
      kst[q] = run;
    }
    __syncthreads();
    // ---- 4. exclusive scan of the even-padded bucket sizes (one bucket per thread); pads
    {
      const int raw = (tid < s) ? kst[tid] : 0;
      const int v = raw + (raw & 1);
      int incl = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) wsum4[wid] = incl;
      __syncthreads();
      int wbase = (lane < wid) ? wsum4[lane] : 0;  // sum of the earlier warps' totals
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) wbase += __shfl_xor_sync(0xffffffffu, wbase, o);
      const int ex = wbase + incl - v;
      if (tid < s) {
        kst[tid] = ex;
        if (raw & 1) ent[ex + raw] = PAD;
      }
      if (tid == S4_THREADS - 1) kst[s] = ex + v;
    }
    __syncthreads();
    // ---- 5. place this thread's entries
    if (valid) {
      const uint32_t eoff = mt_s + (uint32_t)tid * 256u + 8u * s4_g((uint32_t)tid);
#pragma unroll
      for (int t = 0; t < Z; ++t)
        if (t < zeta) {
          const int q = kp[t] & 0xffff;
          ent[kst[q] + cw[wid * NQP + q] + (kp[t] >> 16)] = eoff | (((neg >> t) & 1u) << 31);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- 6. gather: warp-owned buckets, lane = column, two entries per iteration
    {
      int p = (qlo < s) ? kst[qlo] : 0;
#pragma unroll
      for (int i = 0; i < QPW; ++i) {
        const int q = qlo + i;
        if (q < s) {
          const int e = kst[q + 1];
          double t0 = 0.0, t1 = 0.0;
#pragma unroll 1
          for (; p < e; p += 2) {
            const uint2 ee = *reinterpret_cast<const uint2*>(ent + p);
            double x0, x1;  // both loads in flight before either is used
            asm volatile("ld.shared.f64 %0, [%2];\n\tld.shared.f64 %1, [%3];"
                         : "=d"(x0), "=d"(x1)
                         : "r"((ee.x ^ lane8) & amask), "r"((ee.y ^ lane8) & amask));
            t0 += __hiloint2double(__double2hiint(x0) ^ (int)(ee.x & 0x80000000u), __double2loint(x0));
            t1 += __hiloint2double(__double2hiint(x1) ^ (int)(ee.y & 0x80000000u), __double2loint(x1));
          }
          acc[i] += t0 + t1;
        }
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

// out[c*ldo + q] (+)= sum_b part[b][c][q], fixed order: thread group g sums b = g, g+8, ...
// (ascending), then the 8 group sums are added in g order.  32 outputs x 8 groups per CTA.
__global__ void __launch_bounds__(256) sketch_reduce_kernel(const double* __restrict__ part, int grid, int J, int s,
                                                            double* __restrict__ out, int64_t ldo, int accumulate) {
  __shared__ double red[8][33];
  const int l = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t tot = (int64_t)J * s;
  const int64_t o = (int64_t)blockIdx.x * 32 + l;
  double t = 0.0;
  if (o < tot) {
    const double* p = part + o;
#pragma unroll 4
    for (int b = g; b < grid; b += 8) t += p[(int64_t)b * tot];
  }
  red[g][l] = t;
  __syncthreads();
  if (g == 0 && o < tot) {
    double u = red[0][l];
#pragma unroll
    for (int k = 1; k < 8; ++k) u += red[k][l];
    const int c = (int)(o / s), q = (int)(o % s);
    if (accumulate) out[(int64_t)c * ldo + q] += u;
    else out[(int64_t)c * ldo + q] = u;
  }
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

// dynamic shared memory of sketch_v4_kernel for (s, zeta); static part: wsum4
static size_t sketch_v4_smem(int s, int zeta) {
  return 256 + sizeof(double) * (S4_R + 1) * 32 + sizeof(uint32_t) * s4_ent_words(s, zeta) + sizeof(int) * (s + 2) +
         sizeof(uint16_t) * S4_HWARPS * s4_nqp(s) + 16;
}

static bool sketch_v4_fits(int s, int zeta) {
  static int optin = 0;
  if (!optin) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
      cudaGetLastError();
      optin = 232448;
    }
  }
  return s <= S4_QMAX && sketch_v4_smem(s, zeta) + 1024 <= (size_t)optin;
}

template <int QPW, int ZETA>
static cudaError_t launch_v4(const SketchArgs& a, int grid, cudaStream_t st) {
  const size_t smem = sketch_v4_smem(a.s, a.zeta);
  static size_t set = 0;
  if (set < smem) {
    cudaError_t e =
        cudaFuncSetAttribute(sketch_v4_kernel<QPW, ZETA>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return e;
    }
    set = smem;
  }
  sketch_v4_kernel<QPW, ZETA><<<grid, S4_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

template <int ZETA>
static cudaError_t launch_v4_z(const SketchArgs& a, int grid, cudaStream_t st) {
  const int span = a.s;
  if (span <= 8 * S4_WARPS) return launch_v4<8, ZETA>(a, grid, st);
  if (span <= 12 * S4_WARPS) return launch_v4<12, ZETA>(a, grid, st);
  if (span <= 16 * S4_WARPS) return launch_v4<16, ZETA>(a, grid, st);
  if (span <= 20 * S4_WARPS) return launch_v4<20, ZETA>(a, grid, st);
  return launch_v4<24, ZETA>(a, grid, st);
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
  if (sketch_v4_fits(s, zeta)) {
    a.q_base = 0;
    a.tiles = (nrows + S4_R - 1) / S4_R;
    cudaError_t e = (zeta == 8) ? launch_v4_z<8>(a, grid, st) : launch_v4_z<0>(a, grid, st);
    if (e != cudaSuccess) return e;
    if (launches) ++*launches;
    const int64_t tot = (int64_t)J * s;
    sketch_reduce_kernel<<<(int)((tot + 31) / 32), 256, 0, st>>>(part, grid, J, s, out, ldo, accumulate);
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
  sketch_reduce_kernel<<<(int)((tot + 31) / 32), 256, 0, st>>>(part, grid, J, s, out, ldo, accumulate);
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
