// srft.cu -- the SRFT sketch (Eq. SRFT, F = DCT2 as in the paper's experiments,
// P:2041-2043; reading O32):  S x = sqrt(n/s) * DCT2_ortho(E x)[q_0..q_{s-1}].
//
// Per batch of J columns: (1) a pack kernel applies the hashed signs E and the Makhoul reordering
// v = [x_0, x_2, ..., x_3, x_1] (so that DCT2(x)_k = 2 Re(e^{-i pi k/2n} FFT(v)_k)); (2) cuFFT runs a
// batched real-to-complex FFT of length n (the library transform; the only library call on the
// path); (3) a sample kernel evaluates the s sampled DCT coordinates from the half spectrum
// (V_k = conj(V_{n-k}) above n/2), with the orthonormal scaling and sqrt(n/s).  The coordinates
// q_t are drawn on the host by Floyd's algorithm from the same counter hash as the signs.
// Rows are not separable across ranks (the DCT mixes all of them): single-GPU only.
#include <cufft.h>

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

// v[c][j] = E[r] x[c][r] with r = 2j (j < ceil(n/2)) or 2(n-1-j)+1
__global__ void srft_pack_kernel(const double* __restrict__ M, int64_t ldm, int64_t n, int J, uint64_t key,
                                 double* __restrict__ V, int64_t ldv) {
  const int64_t h = (n + 1) / 2;
  const int64_t tot = n * J;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < tot;
       idx += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(idx / n);
    const int64_t j = idx - (int64_t)c * n;
    const int64_t r = (j < h) ? 2 * j : 2 * (n - 1 - j) + 1;
    const uint64_t w = sks_fmix64(key + SKS_GAMMA * (2ull * (uint64_t)r + 1ull));
    const double e = (w & 1ull) ? -1.0 : 1.0;
    V[j + (int64_t)c * ldv] = e * M[r + (int64_t)c * ldm];
  }
}

// out[t + c*ldo] = sqrt(n/s) * ortho * 2 Re(e^{-i pi k / 2n} V_k),  k = q[t]
__global__ void srft_sample_kernel(const double2* __restrict__ Y, int64_t ldy, int64_t n, int J, int s,
                                   const int32_t* __restrict__ q, double* __restrict__ out, int64_t ldo) {
  const int tot = s * J;
  const double sc = sqrt((double)n / (double)s);
  for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += gridDim.x * blockDim.x) {
    const int c = idx / s, t = idx - c * s;
    const int64_t k = q[t];
    const int64_t kk = (k <= n / 2) ? k : n - k;
    double2 V = Y[kk + (int64_t)c * ldy];
    if (k > n / 2) V.y = -V.y;
    double sn, cs;
    sincospi((double)k / (double)(2 * n), &sn, &cs);
    const double X = 2.0 * (V.x * cs + V.y * sn);
    const double ortho = (k == 0) ? sqrt(1.0 / (4.0 * (double)n)) : sqrt(1.0 / (2.0 * (double)n));
    out[t + (int64_t)c * ldo] = sc * ortho * X;
  }
}

struct SrftPlan {  // cuFFT plans by batch width (the batch schedule uses a few widths: 8, 16, 32, ...)
  cufftHandle h[6] = {};
  int64_t n[6] = {};
  int J[6] = {};
  int used = 0;
};

size_t srft_work_doubles(int64_t n, int J) {  // V (n x J) + Y ((n/2+1) x J complex)
  return (size_t)(n + 2) * J + (size_t)2 * (n / 2 + 1) * J + 64;
}

cudaError_t launch_srft(const double* M, int64_t ldm, int64_t n, int J, int s, uint64_t key, const int32_t* q,
                        double* work, void** cache, double* out, int64_t ldo, int num_sms, cudaStream_t st) {
  SrftPlan* p = reinterpret_cast<SrftPlan*>(*cache);
  if (!p) {
    p = new SrftPlan();
    *cache = p;
  }
  const int64_t ldv = (n + 2) & ~int64_t(1);  // even pitch: every column (and the complex output) 16-byte aligned
  double* V = work;
  double2* Y = reinterpret_cast<double2*>(work + (size_t)ldv * J);
  const int64_t ldy = n / 2 + 1;
  int slot = -1;
  for (int i = 0; i < p->used; ++i)
    if (p->n[i] == n && p->J[i] == J) slot = i;
  if (slot < 0) {
    if (p->used == 6) {  // evict all (geometry changed)
      for (int i = 0; i < p->used; ++i) cufftDestroy(p->h[i]);
      p->used = 0;
    }
    slot = p->used;
    long long nn = n, inembed = ldv, onembed = ldy;
    size_t ws = 0;
    if (cufftCreate(&p->h[slot]) != CUFFT_SUCCESS) return cudaErrorUnknown;
    if (cufftMakePlanMany64(p->h[slot], 1, &nn, &inembed, 1, ldv, &onembed, 1, ldy, CUFFT_D2Z, J, &ws) !=
        CUFFT_SUCCESS) {
      cufftDestroy(p->h[slot]);
      return cudaErrorUnknown;
    }
    p->n[slot] = n;
    p->J[slot] = J;
    ++p->used;
  }
  cufftHandle h = p->h[slot];
  const int grid = num_sms * 8;
  srft_pack_kernel<<<grid, 256, 0, st>>>(M, ldm, n, J, key, V, ldv);
  if (cudaGetLastError() != cudaSuccess) return cudaGetLastError();
  if (cufftSetStream(h, st) != CUFFT_SUCCESS) return cudaErrorUnknown;
  if (cufftExecD2Z(h, V, reinterpret_cast<cufftDoubleComplex*>(Y)) != CUFFT_SUCCESS) return cudaErrorUnknown;
  srft_sample_kernel<<<std::max(1, std::min(num_sms * 4, (s * J + 255) / 256)), 256, 0, st>>>(Y, ldy, n, J, s, q,
                                                                                              out, ldo);
  return cudaGetLastError();
}

void srft_free(void* cache) {
  SrftPlan* p = reinterpret_cast<SrftPlan*>(cache);
  if (p)
    for (int i = 0; i < p->used; ++i) cufftDestroy(p->h[i]);
  delete p;
}

}  // namespace sks
