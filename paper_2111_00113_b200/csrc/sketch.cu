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
// v5 (s <= 768): the sketch PLAN is built once per restart cycle (S is fixed within a cycle,
// reading O7), the per-batch kernel only stages the batch and gathers.
//
// Plan of one tile of R = 512 rows: the tile's R*zeta entries bucketed by sketch row q
// (both signs in one bucket), each bucket padded to an even length with an entry pointing at
// a zero row; placement order inside a bucket is (warp, t, lane) from __match_any_sync ranks
// and a prefix over warps -- no atomics, so the plan (and every sum) is bitwise reproducible.
// An entry is E = r*256 + 8*g(r) | sign<<31, the byte offset of row r in the staged tile.
//
// Gather (per batch of J <= 32 columns): Mt[r][c] (R rows + one zero row, 32 columns) lives
// at byte r*256 + 8*(c ^ g(r)), g(r) = r & 31: the staging warp (32 consecutive rows of one
// column, 256 contiguous global bytes) and the gather warp (one row, lane = column) are both
// bank-conflict free and the gather address is one LOP3 ((E ^ 8*lane) & 0x7fffffff).
// 32 warps; warp w owns sketch rows [w*QPW, (w+1)*QPW) with its sums in registers.
// ------------------------------------------------------------------------------
constexpr int S4_R = 512;
constexpr int S4_QMAX = 768;
constexpr int S4_THREADS = 1024;
constexpr int S4_WARPS = S4_THREADS / 32;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src) : "memory");
}
#ifndef SK_PF
#define SK_PF 1
#endif
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
__host__ __device__ __forceinline__ uint32_t s4_g(uint32_t r) { return r & 31u; }
// bulk L2 prefetch of the 16-byte-aligned part of [p, p + bytes) (never outside the range)
__device__ __forceinline__ void l2_prefetch_bulk(const void* p, uint32_t bytes) {
  const uint64_t a = (reinterpret_cast<uint64_t>(p) + 15ull) & ~15ull;
  const uint64_t e = (reinterpret_cast<uint64_t>(p) + bytes) & ~15ull;
  if (e > a) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((uint32_t)(e - a)) : "memory");
}
__host__ __device__ __forceinline__ int s4_nqp(int s) { return (s + 7) & ~7; }
// plan strides: entries (u32) and bucket starts (u16) per tile, both 16-byte multiples
__host__ __device__ __forceinline__ int s5_ent_stride(int s, int zeta) { return (S4_R * zeta + s + 4 + 3) & ~3; }
__host__ __device__ __forceinline__ int s5_kst_stride(int s) { return (s + 1 + 7) & ~7; }

// ---- plan kernel: one CTA per tile (grid-stride), 1024 threads
template <int ZETA>
__global__ void __launch_bounds__(S4_THREADS, 1) sketch_plan_kernel(int64_t nrows, int64_t row_begin, int s,
                                                                     int zeta_rt, uint64_t key, int64_t tiles,
                                                                     uint32_t* __restrict__ pent,
                                                                     uint16_t* __restrict__ pkst) {
  extern __shared__ __align__(16) unsigned char smraw[];
  constexpr int Z = ZETA > 0 ? ZETA : SKS_ZETA_MAX;
  constexpr int ZH = (Z + 1) / 2;  // draws per thread (a row's draws are split over two threads)
  const int zeta = ZETA > 0 ? ZETA : zeta_rt;
  const int zh = (zeta + 1) / 2;
  const int NQP = s4_nqp(s), ES = s5_ent_stride(s, zeta), KS = s5_kst_stride(s);
  uint32_t* ent = reinterpret_cast<uint32_t*>(smraw);       // [ES]
  int* kst = reinterpret_cast<int*>(ent + ES);               // [s + 1]
  uint16_t* cw = reinterpret_cast<uint16_t*>(kst + s + 4);   // [32 warps][NQP]
  uint16_t* qa = cw + S4_WARPS * NQP;                        // [R][ZH]
  __shared__ int wsum4[S4_WARPS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t ltmask = (1u << lane) - 1u;
  const uint32_t PAD = (uint32_t)S4_R * 256u;  // the zero row
  uint16_t* cwm = cw + wid * NQP;
  const int row = tid & (S4_R - 1), half = tid >> 9;  // this thread hashes draws [t0, t1) of `row`
  const int t0 = half ? zh : 0, t1 = half ? zeta : zh;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * S4_R;
    const int nr = (int)((nrows - r0) < (int64_t)S4_R ? (nrows - r0) : (int64_t)S4_R);
    // ---- hash (reading O5)
    for (int i = lane; i < NQP / 2; i += 32) reinterpret_cast<uint32_t*>(cwm)[i] = 0u;
    const bool valid = row < nr;
    const uint64_t hbase = key + SKS_GAMMA * (16ull * (uint64_t)(row_begin + r0 + row));
    int kq[ZH];
    uint32_t neg = 0;
#pragma unroll
    for (int u = 0; u < ZH; ++u) kq[u] = 0;
    if (valid) {
#pragma unroll
      for (int u = 0; u < ZH; ++u) {
        const int t = t0 + u;
        if (t < t1) {
          const uint64_t w = sks_fmix64(hbase + SKS_GAMMA * (uint64_t)(t >> 1));
          const uint32_t uu = (t & 1) ? (uint32_t)(w >> 32) : (uint32_t)(w & 0xffffffffu);
          const uint32_t J = (uint32_t)(s - zeta + t);
          kq[u] = (int)(((uint64_t)uu * (uint64_t)(J + 1u)) >> 32);  // raw draw v_t
        }
      }
      neg = (uint32_t)(sks_fmix64(hbase + SKS_GAMMA * 8ull) & ((1ull << zeta) - 1ull));
      if (half == 0) {  // Floyd among the first-half draws
#pragma unroll
        for (int u = 0; u < ZH; ++u) {
          bool taken = false;
#pragma unroll
          for (int i = 0; i < u; ++i) taken |= (kq[i] == kq[u]);
          if (taken) kq[u] = s - zeta + u;
          if (u < t1) qa[row * ZH + u] = (uint16_t)kq[u];
        }
      }
    }
    __syncthreads();
    if (valid && half == 1) {  // Floyd for the second half against all earlier draws
      int q0[ZH];
#pragma unroll
      for (int i = 0; i < ZH; ++i) q0[i] = (i < zh) ? (int)qa[row * ZH + i] : -1;
#pragma unroll
      for (int u = 0; u < ZH; ++u) {
        bool taken = false;
#pragma unroll
        for (int i = 0; i < ZH; ++i) taken |= (q0[i] == kq[u]);
#pragma unroll
        for (int i = 0; i < u; ++i) taken |= (kq[i] == kq[u]);
        if (taken) kq[u] = s - zeta + t0 + u;
      }
    }
    // ---- per-warp ranks per bucket q (warp slot = wid)
#pragma unroll
    for (int u = 0; u < ZH; ++u) {
      const int t = t0 + u;
      const int k = (valid && t < t1) ? kq[u] : -1 - lane;
      const uint32_t mm = __match_any_sync(0xffffffffu, k);
      const int base = (k >= 0) ? (int)cwm[k] : 0;
      kq[u] = (k & 0xffff) | ((base + __popc(mm & ltmask)) << 16);
      __syncwarp();
      if (k >= 0 && (mm & ltmask) == 0u) cwm[k] = (uint16_t)(base + __popc(mm));
      __syncwarp();
    }
    __syncthreads();
    // ---- per-bucket prefix over the 32 warp slots (cw := warp offset in the bucket)
    for (int q = tid; q < s; q += S4_THREADS) {
      int run = 0;
#pragma unroll 8
      for (int w = 0; w < S4_WARPS; ++w) {
        const int c = cw[w * NQP + q];
        cw[w * NQP + q] = (uint16_t)run;
        run += c;
      }
      kst[q] = run;
    }
    __syncthreads();
    // ---- exclusive scan of the even-padded bucket sizes (one bucket per thread); pads
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
    // ---- place this thread's entries
    if (valid) {
      const uint32_t eoff = (uint32_t)row * 256u + 8u * s4_g((uint32_t)row);
#pragma unroll
      for (int u = 0; u < ZH; ++u) {
        const int t = t0 + u;
        if (t < t1) {
          const int q = kq[u] & 0xffff;
          ent[kst[q] + cwm[q] + (kq[u] >> 16)] = eoff | (((neg >> t) & 1u) << 31);
        }
      }
    }
    __syncthreads();
    // ---- write the plan of this tile
    const int ne = kst[s];
    uint32_t* ge = pent + tile * (int64_t)ES;
    for (int i = tid; i < ne; i += S4_THREADS) ge[i] = ent[i];
    uint16_t* gk = pkst + tile * (int64_t)KS;
    for (int i = tid; i < KS; i += S4_THREADS) gk[i] = (uint16_t)(i <= s ? kst[i] : ne);
    __syncthreads();
  }
}

// ---- gather kernel: stage the batch + load the tile plan (cp.async), gather
// LPE = lanes per plan entry (32 for J > 16).  A batch of J <= 16 (<= 8) columns is gathered by half- (quarter-)
// warps: lane = (entry slot, column), so one warp instruction moves 2 (4) entries and a narrow batch costs
// proportionally fewer shared-memory wavefronts (a half-row of 16 columns of Mt covers the 32 banks once, whatever
// its swizzle); each lane's sums are partial over its entry slot and are combined by a fixed shuffle at the end.
template <int QPW, int LPE>
__global__ void __launch_bounds__(S4_THREADS, 1) sketch_v5_kernel(SketchArgs a, const uint32_t* __restrict__ pent,
                                                                  const uint16_t* __restrict__ pkst, int ES, int KS) {
  constexpr int EPI = 32 / LPE;  // entries per warp instruction
  extern __shared__ __align__(16) unsigned char smraw[];
  const int s = a.s;
  double* Mt = reinterpret_cast<double*>(smraw);                   // [(R+1)*32]
  uint32_t* ent = reinterpret_cast<uint32_t*>(Mt + (S4_R + 1) * 32);  // [ES]
  uint16_t* kst = reinterpret_cast<uint16_t*>(ent + ES);             // [KS]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t lane8, amask;  // opaque to the optimiser (keeps the gather address a single LOP3)
  asm("mov.b32 %0, %1;" : "=r"(lane8) : "r"((uint32_t)(lane % LPE) * 8u));
  const int slot_e = lane / LPE;  // entry slot of this lane
  asm("mov.b32 %0, %1;" : "=r"(amask) : "r"(0x7fffffffu));
  const uint32_t mt_s = smem_addr(Mt), ent_s = smem_addr(ent), kst_s = smem_addr(kst);
  const int qlo = wid * QPW;
  const uint32_t st_base = mt_s + (uint32_t)lane * 256u + 8u * ((uint32_t)(wid ^ lane) & 31u);
  if (tid < 32) Mt[S4_R * 32 + tid] = 0.0;

  double acc[QPW];
#pragma unroll
  for (int i = 0; i < QPW; ++i) acc[i] = 0.0;

  const int64_t t_lo = (a.tiles * blockIdx.x) / gridDim.x;
  const int64_t t_hi = (a.tiles * (blockIdx.x + 1)) / gridDim.x;
  for (int64_t tile = t_lo; tile < t_hi; ++tile) {
    const int64_t r0 = tile * S4_R;
    const int nr = (int)((a.nrows - r0) < (int64_t)S4_R ? (a.nrows - r0) : (int64_t)S4_R);
    // ---- stage: warp w moves column w (32 consecutive rows per instruction)
    if (wid < a.J) {
      const double* src = a.M + (int64_t)wid * a.ldm + r0 + lane;
      if (nr == S4_R) {
#pragma unroll
        for (int i = 0; i < S4_R / 32; ++i) cp_async8(st_base + i * 8192u, src + i * 32);
      } else {
        for (int i = 0; i < S4_R / 32; ++i)
          if (i * 32 + lane < nr) cp_async8(st_base + i * 8192u, src + i * 32);
      }
    }
    // ---- the tile's plan (16-byte chunks)
    {
      const uint32_t* ge = pent + tile * (int64_t)ES;
      for (int i = tid; i < ES / 4; i += S4_THREADS) cp_async16(ent_s + 16u * i, ge + 4 * i);
      const uint16_t* gk = pkst + tile * (int64_t)KS;
      for (int i = tid; i < KS / 8; i += S4_THREADS) cp_async16(kst_s + 16u * i, gk + 8 * i);
    }
    cp_async_wait_all();
    __syncthreads();
    // ---- pull the next tile (its J column segments and its plan) into L2 while this one is
    //      gathered, so that the next staging is served from L2 instead of HBM
    if (wid == 0 && tile + 1 < t_hi) {
      const int64_t rn = r0 + S4_R;
      const int nrn = (int)((a.nrows - rn) < (int64_t)S4_R ? (a.nrows - rn) : (int64_t)S4_R);
      if (lane < a.J) l2_prefetch_bulk(a.M + (int64_t)lane * a.ldm + rn, (uint32_t)(nrn * 8));
      if (lane == 31) l2_prefetch_bulk(pent + (tile + 1) * (int64_t)ES, (uint32_t)(ES * 4));
    }
    // ---- gather: warp-owned buckets, lane = column, two entries per iteration; the bucket
    //      boundaries of the warp come from one load + shuffles
    {
      const int kb = (lane <= QPW) ? (int)kst[min(qlo + lane, s)] : 0;
      int p = __shfl_sync(0xffffffffu, kb, 0);
      // SK_PF: the next entry pair is loaded one iteration ahead (the warp's buckets are contiguous in ent[], and
      // ent[] extends past the last bucket), so the gather's two dependent shared loads overlap
      uint2 eenx = (SK_PF && LPE == 32) ? *reinterpret_cast<const uint2*>(ent + p) : make_uint2(0u, 0u);
#pragma unroll
      for (int i = 0; i < QPW; ++i) {
        const int e = __shfl_sync(0xffffffffu, kb, i + 1);
        double t0a = 0.0, t1a = 0.0;
        if constexpr (LPE < 32) {
          // EPI entries per instruction; entries past the bucket end read the zero row (offset R*256)
#pragma unroll 1
          for (; p < e; p += 2 * EPI) {
            const int i0 = p + slot_e, i1 = p + EPI + slot_e;
            const uint32_t e0 = (EPI == 2 || i0 < e) ? ent[i0] : (uint32_t)S4_R * 256u;
            const uint32_t e1 = (i1 < e) ? ent[i1] : (uint32_t)S4_R * 256u;
            double x0, x1;
            uint32_t o0, o1;
            asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(o0) : "r"(e0), "r"(lane8), "r"(amask));
            asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(o1) : "r"(e1), "r"(lane8), "r"(amask));
            asm volatile("ld.shared.f64 %0, [%2];\n\tld.shared.f64 %1, [%3];"
                         : "=d"(x0), "=d"(x1)
                         : "r"(mt_s + o0), "r"(mt_s + o1));
            t0a += __hiloint2double(__double2hiint(x0) ^ (int)(e0 & 0x80000000u), __double2loint(x0));
            t1a += __hiloint2double(__double2hiint(x1) ^ (int)(e1 & 0x80000000u), __double2loint(x1));
          }
          p = e;
        } else
#pragma unroll 1
        for (; p < e; p += 2) {
#if SK_PF
          const uint2 ee = eenx;
          eenx = *reinterpret_cast<const uint2*>(ent + p + 2);
#else
          const uint2 ee = *reinterpret_cast<const uint2*>(ent + p);
#endif
          double x0, x1;  // both loads in flight before either is used
          uint32_t o0, o1;  // (E ^ 8 lane) & 0x7fffffff as one LOP3 each
          asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(o0) : "r"(ee.x), "r"(lane8), "r"(amask));
          asm("lop3.b32 %0, %1, %2, %3, 0x28;" : "=r"(o1) : "r"(ee.y), "r"(lane8), "r"(amask));
          asm volatile("ld.shared.f64 %0, [%2];\n\tld.shared.f64 %1, [%3];"
                       : "=d"(x0), "=d"(x1)
                       : "r"(mt_s + o0), "r"(mt_s + o1));
          t0a += __hiloint2double(__double2hiint(x0) ^ (int)(ee.x & 0x80000000u), __double2loint(x0));
          t1a += __hiloint2double(__double2hiint(x1) ^ (int)(ee.y & 0x80000000u), __double2loint(x1));
        }
        acc[i] += t0a + t1a;
      }
    }
    __syncthreads();
  }
  if constexpr (LPE < 32) {  // combine the entry slots' partial sums (fixed order)
#pragma unroll
    for (int i = 0; i < QPW; ++i) {
#pragma unroll
      for (int o = 16; o >= LPE; o >>= 1) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
    }
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
  cudaError_t e = set_smem_attr(sketch_batch_kernel<QPW, ZETA>, smem);
  if (e != cudaSuccess) return e;
  sketch_batch_kernel<QPW, ZETA><<<grid, SK_THREADS, smem, st>>>(a);
  return cudaGetLastError();
}

static int sm_optin() {
  static int optin = 0;
  if (!optin) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
      cudaGetLastError();
      optin = 232448;
    }
  }
  return optin;
}

static size_t sketch_plan_smem(int s, int zeta) {
  return sizeof(uint32_t) * s5_ent_stride(s, zeta) + sizeof(int) * (s + 4) + sizeof(uint16_t) * S4_WARPS * s4_nqp(s) +
         sizeof(uint16_t) * S4_R * 8 + 16;
}
static size_t sketch_v5_smem(int s, int zeta) {
  return sizeof(double) * (S4_R + 1) * 32 + sizeof(uint32_t) * s5_ent_stride(s, zeta) +
         sizeof(uint16_t) * s5_kst_stride(s) + 16;
}

bool sketch_plan_supported(int s, int zeta) {
  return s <= S4_QMAX && zeta <= SKS_ZETA_MAX && sketch_v5_smem(s, zeta) + 1024 <= (size_t)sm_optin() &&
         sketch_plan_smem(s, zeta) + 1024 <= (size_t)sm_optin();
}

size_t sketch_plan_bytes(int64_t nrows, int s, int zeta) {
  const int64_t tiles = (nrows + S4_R - 1) / S4_R;
  return (size_t)tiles * (sizeof(uint32_t) * s5_ent_stride(s, zeta) + sizeof(uint16_t) * s5_kst_stride(s));
}

template <typename K>
static cudaError_t set_smem(K kern, size_t smem) {
  return set_smem_attr(kern, smem);
}

cudaError_t launch_sketch_plan(int64_t nrows, int64_t row_begin, int s, int zeta, uint64_t key, void* plan,
                               int num_sms, cudaStream_t st) {
  if (!sketch_plan_supported(s, zeta)) return cudaErrorInvalidValue;
  const int64_t tiles = (nrows + S4_R - 1) / S4_R;
  uint32_t* pent = reinterpret_cast<uint32_t*>(plan);
  uint16_t* pkst = reinterpret_cast<uint16_t*>(pent + tiles * (int64_t)s5_ent_stride(s, zeta));
  const size_t smem = sketch_plan_smem(s, zeta);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, (int64_t)num_sms * 2));
  cudaError_t e;
  if (zeta == 8) {
    if ((e = set_smem(sketch_plan_kernel<8>, smem)) != cudaSuccess) return e;
    sketch_plan_kernel<8><<<grid, S4_THREADS, smem, st>>>(nrows, row_begin, s, zeta, key, tiles, pent, pkst);
  } else {
    if ((e = set_smem(sketch_plan_kernel<0>, smem)) != cudaSuccess) return e;
    sketch_plan_kernel<0><<<grid, S4_THREADS, smem, st>>>(nrows, row_begin, s, zeta, key, tiles, pent, pkst);
  }
  return cudaGetLastError();
}

template <int QPW, int LPE>
static cudaError_t launch_v5l(const SketchArgs& a, const void* plan, int grid, cudaStream_t st) {
  const size_t smem = sketch_v5_smem(a.s, a.zeta);
  cudaError_t e = set_smem(sketch_v5_kernel<QPW, LPE>, smem);
  if (e != cudaSuccess) return e;
  const int ES = s5_ent_stride(a.s, a.zeta), KS = s5_kst_stride(a.s);
  const uint32_t* pent = reinterpret_cast<const uint32_t*>(plan);
  const uint16_t* pkst = reinterpret_cast<const uint16_t*>(pent + a.tiles * (int64_t)ES);
  sketch_v5_kernel<QPW, LPE><<<grid, S4_THREADS, smem, st>>>(a, pent, pkst, ES, KS);
  return cudaGetLastError();
}

static int sketch_narrow() {  // SKS_SKETCH_NARROW=0: every batch gathered with 32 lanes per entry (A/B)
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("SKS_SKETCH_NARROW");
    v = e ? (e[0] != '0') : 1;
  }
  return v;
}

template <int QPW>
static cudaError_t launch_v5(const SketchArgs& a, const void* plan, int grid, cudaStream_t st) {
  if (sketch_narrow() && a.J <= 8) return launch_v5l<QPW, 8>(a, plan, grid, st);
  if (sketch_narrow() && a.J <= 16) return launch_v5l<QPW, 16>(a, plan, grid, st);
  return launch_v5l<QPW, 32>(a, plan, grid, st);
}

static cudaError_t launch_v5_q(const SketchArgs& a, const void* plan, int grid, cudaStream_t st) {
  const int span = a.s;
  if (span <= 8 * S4_WARPS) return launch_v5<8>(a, plan, grid, st);
  if (span <= 12 * S4_WARPS) return launch_v5<12>(a, plan, grid, st);
  if (span <= 16 * S4_WARPS) return launch_v5<16>(a, plan, grid, st);
  if (span <= 20 * S4_WARPS) return launch_v5<20>(a, plan, grid, st);
  return launch_v5<24>(a, plan, grid, st);
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
                          int accumulate, cudaStream_t st, int64_t* launches, const void* plan) {
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
  if (plan != nullptr) {
    if (!sketch_plan_supported(s, zeta)) return cudaErrorInvalidValue;
    a.q_base = 0;
    a.tiles = (nrows + S4_R - 1) / S4_R;
    cudaError_t e = launch_v5_q(a, plan, grid, st);
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
