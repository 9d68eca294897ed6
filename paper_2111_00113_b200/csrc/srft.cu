// srft.cu -- the SRFT sketch (Eq. SRFT, F = DCT2 as in the paper's experiments,
// P:2041-2043; reading O32):  S x = sqrt(n/s) * DCT2_ortho(E x)[q_0..q_{s-1}].
//
// Only s of the n DCT coordinates are ever used, so the transform is a hand-written OUTPUT-PRUNED DFT (no FFT
// library): with the Makhoul reordering v = [x_0, x_2, ..., x_3, x_1] (sign-flipped by the hashed E),
// DCT2(x)_k = 2 Re(e^{-i pi k/2n} Y_k), Y_k = sum_j v_j e^{-2 pi i jk/n}, and with n = n1 n2 (n1 the largest
// divisor of n not above 32), j = n2 j1 + j2:
//     Y_k = sum_{j2 < n2} e^{-2 pi i k j2/n} Z_{j2}(k mod n1),   Z_{j2}(q) = sum_{j1 < n1} v_{n2 j1 + j2} w1^{q j1}
// (w1 = e^{-2 pi i/n1}).  Per batch of J columns:
//   (1) srft_stage1_kernel: one thread per (j2, column) gathers its n1 reordered, signed entries of x and forms
//       the n1-point DFT Z_{j2}(q) for every q (direct, twiddle table in shared memory);
//   (2) srft_stage2_kernel: for the sampled k grouped by q = k mod n1 (srft_group_kernel), a complex
//       (k x j2) . (j2 x column) contraction per group, twiddles e^{-2 pi i k j2/n} from the exact integer phase
//       (k j2 mod n) staged in shared memory, split over j2 chunks (partial sums per chunk);
//   (3) srft_finish_kernel: the chunk partials summed in a fixed order, DCT coordinate and orthonormal scaling
//       sqrt(n/s) * ortho_k * 2 Re(e^{-i pi k/2n} Y_k).
// Cost per column ~ n (n1 + s/n1) complex multiply-adds instead of a full FFT's n log n passes over memory;
// deterministic (fixed summation orders).  The coordinates q_t are drawn on the host by Floyd's algorithm from
// the same counter hash as the signs.  Rows are not separable across ranks (the DCT mixes all of them):
// single-GPU only.
#include <unordered_set>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace sks {

static constexpr uint64_t SRFT_DOMAIN = 0x5352465444435432ull;

static uint64_t host_fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}

uint64_t srft_key_host(uint64_t seed, uint32_t cycle) {
  return host_fmix64(host_fmix64(seed ^ SRFT_DOMAIN) + 0x9E3779B97F4A7C15ull * (uint64_t)(cycle + 1));
}

void srft_rows_host(int64_t n, int s, uint64_t key, int32_t* q) {
  std::unordered_set<int64_t> taken;
  taken.reserve((size_t)s * 2);
  for (int t = 0; t < s; ++t) {
    const uint64_t u = host_fmix64(key + 0x9E3779B97F4A7C15ull * (2ull * (uint64_t)t + 2ull)) & 0xFFFFFFFFull;
    const int64_t J = n - s + t;
    int64_t v = (int64_t)((u * (uint64_t)(J + 1)) >> 32);
    if (taken.count(v)) v = J;
    taken.insert(v);
    q[t] = (int32_t)v;
  }
}


constexpr int SR_N1MAX = 32;   // stage-1 DFT length bound
constexpr int SR_TG = 32;      // sampled k per stage-2 sub-group
constexpr int SR_JT = 32;      // j2 per stage-2 tile
constexpr int SR_KC = 4096;    // j2 per stage-2 split (partial sums per split)
constexpr int SR_T2 = 128;     // stage-2 threads: 16 k-pairs x 8 column-quads

static int srft_n1(int64_t n) {
  for (int d = SR_N1MAX; d >= 1; --d)
    if (n % d == 0) return d;
  return 1;
}

__host__ __device__ constexpr int brev5(int j) {
  return ((j & 1) << 4) | ((j & 2) << 2) | (j & 4) | ((j & 8) >> 2) | ((j & 16) >> 4);
}
// one radix-2 stage of the 32-point DIT FFT: butterflies of span LEN, twiddles w^(k 32/LEN), w = e^{-2 pi i/32}
template <int LEN>
__device__ __forceinline__ void fft32_stage(double (&re)[32], double (&im)[32], const double2* tw) {
  constexpr int H = LEN / 2;
#pragma unroll
  for (int i = 0; i < 32; i += LEN)
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const double2 w = tw[k * (32 / LEN)];
      const double tr = re[i + k + H] * w.x - im[i + k + H] * w.y;
      const double ti = re[i + k + H] * w.y + im[i + k + H] * w.x;
      re[i + k + H] = re[i + k] - tr;
      im[i + k + H] = im[i + k] - ti;
      re[i + k] += tr;
      im[i + k] += ti;
    }
}

// Z[c][q][j2] (complex) = sum_{j1 < n1} v_{n2 j1 + j2} w1^{q j1},  v_j = E[r] x[r], r = 2j or 2(n-1-j)+1
__global__ void __launch_bounds__(256, 2) srft_stage1_kernel(const double* __restrict__ M, int64_t ldm, int64_t n,
                                                          int n1, int64_t n2, uint64_t key, double2* __restrict__ Z) {
  __shared__ double2 tw[SR_N1MAX];
  if (threadIdx.x < n1) {
    double sn, cs;
    sincospi(2.0 * (double)threadIdx.x / (double)n1, &sn, &cs);
    tw[threadIdx.x] = make_double2(cs, -sn);  // w1^t
  }
  __syncthreads();
  const int c = blockIdx.y;
  const int64_t j2 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j2 >= n2) return;
  const int64_t h = (n + 1) / 2;
  const double* x = M + (int64_t)c * ldm;
  double v[SR_N1MAX];
#pragma unroll
  for (int j1 = 0; j1 < SR_N1MAX; ++j1) {
    if (j1 < n1) {
      const int64_t j = n2 * j1 + j2;
      const int64_t r = (j < h) ? 2 * j : 2 * (n - 1 - j) + 1;
      const uint64_t w = sks_fmix64(key + SKS_GAMMA * (2ull * (uint64_t)r + 1ull));
      v[j1] = (w & 1ull) ? -x[r] : x[r];
    } else {
      v[j1] = 0.0;
    }
  }
  double2* z = Z + ((int64_t)c * n1) * n2 + j2;
  if (n1 == 32) {  // radix-2 decimation-in-time FFT in registers (input in bit-reversed order)
    double re[32], im[32];
#pragma unroll
    for (int j1 = 0; j1 < 32; ++j1) {
      re[brev5(j1)] = v[j1];
      im[brev5(j1)] = 0.0;
    }
    fft32_stage<2>(re, im, tw);
    fft32_stage<4>(re, im, tw);
    fft32_stage<8>(re, im, tw);
    fft32_stage<16>(re, im, tw);
    fft32_stage<32>(re, im, tw);
#pragma unroll
    for (int q = 0; q < 32; ++q) z[(int64_t)q * n2] = make_double2(re[q], im[q]);
    return;
  }
  for (int q = 0; q < n1; ++q) {
    double re = 0.0, im = 0.0;
    int e = 0;  // (q j1) mod n1
#pragma unroll
    for (int j1 = 0; j1 < SR_N1MAX; ++j1) {
      if (j1 < n1) {
        const double2 t = tw[e];
        re = fma(v[j1], t.x, re);
        im = fma(v[j1], t.y, im);
        e += q;
        if (e >= n1) e -= n1;
      }
    }
    z[(int64_t)q * n2] = make_double2(re, im);
  }
}

// group the s sampled coordinates by q = k mod n1 (counting sort, stable in t): perm[], start[n1 + 1]
__global__ void srft_group_kernel(const int32_t* __restrict__ qk, int s, int n1, int* __restrict__ perm,
                                  int* __restrict__ start) {
  if (threadIdx.x != 0) return;
  for (int q = 0; q <= n1; ++q) start[q] = 0;
  for (int t = 0; t < s; ++t) ++start[qk[t] % n1 + 1];
  for (int q = 0; q < n1; ++q) start[q + 1] += start[q];
  int fill[SR_N1MAX];
  for (int q = 0; q < n1; ++q) fill[q] = start[q];
  for (int t = 0; t < s; ++t) perm[fill[qk[t] % n1]++] = t;
}

// partial Y over one j2 chunk for the sampled k of group q: part[chunk][t][c] (complex)
__global__ void __launch_bounds__(SR_T2) srft_stage2_kernel(const double2* __restrict__ Z, int64_t n, int n1,
                                                            int64_t n2, int J, int s, const int32_t* __restrict__ qk,
                                                            const int* __restrict__ perm, const int* __restrict__ start,
                                                            double2* __restrict__ part) {
  extern __shared__ __align__(16) unsigned char sr_sm[];
  double2(*Zs)[33] = reinterpret_cast<double2(*)[33]>(sr_sm);                              // [j2][c]
  double2(*Ts)[SR_JT + 1] = reinterpret_cast<double2(*)[SR_JT + 1]>(sr_sm + sizeof(double2) * SR_JT * 33);
  double2(*Ps)[SR_JT] = reinterpret_cast<double2(*)[SR_JT]>(sr_sm + sizeof(double2) * (SR_JT * 33 + SR_TG * (SR_JT + 1)));
  __shared__ int64_t ks[SR_TG];
  __shared__ double2 Bs[SR_TG];
  const int q = blockIdx.y;
  const int chunk = blockIdx.x;
  const int64_t jb = (int64_t)chunk * SR_KC, je = (n2 < jb + SR_KC) ? n2 : jb + SR_KC;
  const int g0 = start[q], g1 = start[q + 1];
  const int tid = threadIdx.x;
  const int tp = tid >> 3, cq = tid & 7;  // k pair tp (k = 2 tp, 2 tp + 1), columns cq + 8 b (b < 4): a warp's
                                          // 8 column lanes read 8 consecutive double2 (conflict-free)
  for (int sg = g0; sg < g1; sg += SR_TG) {
    const int G = min(SR_TG, g1 - sg);
    if (tid < G) ks[tid] = qk[perm[sg + tid]];
    __syncthreads();
    for (int i = tid; i < G * SR_JT; i += SR_T2) {  // P[k][jj] = e^{-2 pi i k jj/n}, exact, once per group
      const int kk = i / SR_JT, jj = i - kk * SR_JT;
      double sn, cs;
      sincospi(2.0 * (double)(((uint64_t)ks[kk] * (uint64_t)jj) % (uint64_t)n) / (double)n, &sn, &cs);
      Ps[kk][jj] = make_double2(cs, -sn);
    }
    double2 acc[2][4];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b] = make_double2(0.0, 0.0);
    for (int64_t j0 = jb; j0 < je; j0 += SR_JT) {
      const int L = (int)((je - j0 < SR_JT) ? je - j0 : SR_JT);
      __syncthreads();  // ks visible; the previous tile consumed
      for (int i = tid; i < L * 32; i += SR_T2) {  // Z tile (zero for absent columns), contiguous j2 per warp
        const int c = i / L, jj = i - c * L;
        Zs[jj][c] = (c < J) ? Z[((int64_t)c * n1 + q) * n2 + j0 + jj] : make_double2(0.0, 0.0);
      }
      if (tid < G) {  // the tile's base twiddle e^{-2 pi i k j0/n} from the exact integer phase (< 2^62)
        double sn, cs;
        sincospi(2.0 * (double)(((uint64_t)ks[tid] * (uint64_t)j0) % (uint64_t)n) / (double)n, &sn, &cs);
        Bs[tid] = make_double2(cs, -sn);
      }
      __syncthreads();
      for (int i = tid; i < G * L; i += SR_T2) {  // T[k][jj] = base_k P[k][jj]: one rounding per entry
        const int kk = i / L, jj = i - kk * L;
        const double2 b = Bs[kk], p = Ps[kk][jj];
        Ts[kk][jj] = make_double2(b.x * p.x - b.y * p.y, fma(b.x, p.y, b.y * p.x));
      }
      __syncthreads();
      if (2 * tp < G && cq < J) {
        for (int jj = 0; jj < L; ++jj) {
          double2 t[2], zc[4];
#pragma unroll
          for (int a = 0; a < 2; ++a) t[a] = Ts[min(2 * tp + a, SR_TG - 1)][jj];
#pragma unroll
          for (int b = 0; b < 4; ++b) zc[b] = Zs[jj][cq + 8 * b];
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              acc[a][b].x = fma(t[a].x, zc[b].x, fma(-t[a].y, zc[b].y, acc[a][b].x));
              acc[a][b].y = fma(t[a].x, zc[b].y, fma(t[a].y, zc[b].x, acc[a][b].y));
            }
        }
      }
    }
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int kk = 2 * tp + a, c = cq + 8 * b;
        if (kk < G && c < J) part[((int64_t)chunk * s + perm[sg + kk]) * J + c] = acc[a][b];
      }
  }
}

// out[t + c ldo] = sqrt(n/s) ortho_k 2 Re(e^{-i pi k/2n} Y_k),  Y = sum over the chunks in order
__global__ void srft_finish_kernel(const double2* __restrict__ part, int nchunk, int64_t n, int J, int s,
                                   const int32_t* __restrict__ qk, double* __restrict__ out, int64_t ldo) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= s * J) return;
  const int t = idx / J, c = idx - t * J;
  double yr = 0.0, yi = 0.0;
  for (int ch = 0; ch < nchunk; ++ch) {
    const double2 p = part[((int64_t)ch * s + t) * J + c];
    yr += p.x;
    yi += p.y;
  }
  const int64_t k = qk[t];
  double sn, cs;
  sincospi((double)k / (double)(2 * n), &sn, &cs);
  const double X = 2.0 * (yr * cs + yi * sn);
  const double ortho = (k == 0) ? sqrt(1.0 / (4.0 * (double)n)) : sqrt(1.0 / (2.0 * (double)n));
  out[t + (int64_t)c * ldo] = sqrt((double)n / (double)s) * ortho * X;
}

size_t srft_work_doubles(int64_t n, int J) {  // Z (n x J complex) + chunk partials + grouping
  const int64_t n2 = n / srft_n1(n);
  const int64_t nchunk = (n2 + SR_KC - 1) / SR_KC;
  return (size_t)2 * n * J + (size_t)2 * nchunk * SKS_SMAX * J + SKS_SMAX + SR_N1MAX + 64;
}

cudaError_t launch_srft(const double* M, int64_t ldm, int64_t n, int J, int s, uint64_t key, const int32_t* q,
                        double* work, void** cache, double* out, int64_t ldo, int num_sms, cudaStream_t st) {
  (void)cache;
  (void)num_sms;
  if (J < 1 || J > 32 || s < 1 || s > SKS_SMAX) return cudaErrorInvalidValue;
  const int n1 = srft_n1(n);
  const int64_t n2 = n / n1;
  const int nchunk = (int)((n2 + SR_KC - 1) / SR_KC);
  double2* Z = reinterpret_cast<double2*>(work);
  double2* part = Z + (size_t)n * J;
  int* perm = reinterpret_cast<int*>(part + (size_t)nchunk * SKS_SMAX * J);
  int* start = perm + SKS_SMAX;
  srft_stage1_kernel<<<dim3((unsigned)((n2 + 255) / 256), (unsigned)J), 256, 0, st>>>(M, ldm, n, n1, n2, key, Z);
  srft_group_kernel<<<1, 32, 0, st>>>(q, s, n1, perm, start);
  const size_t sm2 = sizeof(double2) * (SR_JT * 33 + SR_TG * (SR_JT + 1) + SR_TG * SR_JT);
  if (cudaError_t e = set_smem_attr(srft_stage2_kernel, sm2)) return e;
  srft_stage2_kernel<<<dim3((unsigned)nchunk, (unsigned)n1), SR_T2, sm2, st>>>(Z, n, n1, n2, J, s, q, perm, start,
                                                                               part);
  srft_finish_kernel<<<(s * J + 255) / 256, 256, 0, st>>>(part, nchunk, n, J, s, q, out, ldo);
  return cudaGetLastError();
}

void srft_free(void* cache) { (void)cache; }

}  // namespace sks
