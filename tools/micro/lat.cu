// Latency microbenchmark (one warp): dependent chains of DFMA, DMUL, rsqrt.approx.f64, shared
// round trip (STS -> syncwarp -> LDS), shfl.  Prints cycles per operation.
#include <cstdio>
__global__ void lat(double* out, long long* cyc, double a, double b) {
  __shared__ double sm[64];
  const int lane = threadIdx.x;
  double x = a + lane;
  long long t0 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = fma(x, b, a);
  long long t1 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x * b;
  long long t2 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); x = y; }
  long long t3 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) { sm[lane] = x; __syncwarp(); x = sm[(lane + 1) & 31]; __syncwarp(); }
  long long t4 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = __shfl_sync(0xffffffffu, x, (lane + 1) & 31);
  long long t5 = clock64();
#pragma unroll 1
  for (int i = 0; i < 1000; ++i) x = x + b;
  long long t6 = clock64();
  out[lane] = x;
  if (lane == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5; }
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 256); cudaMallocManaged(&c, 64);
  for (int r = 0; r < 2; ++r) { lat<<<1, 32>>>(o, c, 1.0000001, 0.9999999); cudaDeviceSynchronize(); }
  const char* nm[] = {"dfma", "dmul", "rsqrt.approx.f64", "sts+syncwarp+lds+syncwarp", "shfl.f64", "dadd"};
  for (int i = 0; i < 6; ++i) printf("%-28s %.1f cycles/op (incl. loop overhead)\n", nm[i], c[i] / 1000.0);
  return 0;
}
