// Standalone check of jacobi_svd_kernel and small_gemm_kernel (nvcc -I csrc svd_check.cu csrc/svd.cu).
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
namespace sks {
cudaError_t launch_jacobi_svd(const double* M, int ldm, int rows, int n, double tol, int max_sweeps, double* work,
                              double* sigma, double* Ut, double* Vs, int* out, cudaStream_t st);
cudaError_t launch_small_gemm(int M, int N, int K, const double* A, int lda, int ta, const double* B, int ldb,
                              int tb, const double* rs, int rs_inv, double* C, int ldc, cudaStream_t st);
}
int main(int argc, char** argv) {
  const int rows = argc > 1 ? atoi(argv[1]) : 80, n = argc > 2 ? atoi(argv[2]) : 40;
  std::vector<double> M((size_t)rows * n);
  srand(1);
  for (auto& v : M) v = (double)rand() / RAND_MAX - 0.5;
  double *dM, *dw, *ds, *dU, *dV, *dC;
  int* dout;
  cudaMalloc(&dM, 8 * M.size());
  cudaMalloc(&dw, 8 * ((size_t)rows * n + (size_t)n * n + n + 16));
  cudaMalloc(&ds, 8 * (n + 64));
  cudaMalloc(&dU, 8 * (size_t)rows * n);
  cudaMalloc(&dV, 8 * (size_t)n * n);
  cudaMalloc(&dC, 8 * (size_t)rows * n);
  cudaMalloc(&dout, 16);
  cudaMemcpy(dM, M.data(), 8 * M.size(), cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    int st = (int)sks::launch_jacobi_svd(dM, rows, rows, n, 1e14, 60, dw, ds, dU, dV, dout, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("svd launch %d  %.3f ms  sync %s\n", st, ms, cudaGetErrorString(cudaDeviceSynchronize()));
  }
  int out[3];
  cudaMemcpy(out, dout, 12, cudaMemcpyDeviceToHost);
  std::vector<double> s(n), U((size_t)rows * n), V((size_t)n * n);
  cudaMemcpy(s.data(), ds, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(U.data(), dU, 8 * U.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(V.data(), dV, 8 * V.size(), cudaMemcpyDeviceToHost);
  printf("rank %d sweeps %d conv %d  sigma %.6f %.6f ... %.6f\n", out[0], out[1], out[2], s[0], s[1], s[n - 1]);
  // reconstruction error || M - U S V^T ||_max, orthogonality of U and V
  double er = 0, eu = 0, ev = 0;
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < n; ++j) {
      double a = 0;
      for (int k = 0; k < n; ++k) a += U[i + (size_t)k * rows] * s[k] * V[j + (size_t)k * n];
      er = fmax(er, fabs(a - M[i + (size_t)j * rows]));
    }
  for (int a = 0; a < n; ++a)
    for (int b = 0; b < n; ++b) {
      double x = 0, y = 0;
      for (int i = 0; i < rows; ++i) x += U[i + (size_t)a * rows] * U[i + (size_t)b * rows];
      for (int i = 0; i < n; ++i) y += V[i + (size_t)a * n] * V[i + (size_t)b * n];
      eu = fmax(eu, fabs(x - (a == b)));
      ev = fmax(ev, fabs(y - (a == b)));
    }
  printf("recon %.3e  UtU-I %.3e  VtV-I %.3e\n", er, eu, ev);
  // gemm check: C = U^T M (n x n) vs S V^T
  sks::launch_small_gemm(n, n, rows, dU, rows, 1, dM, rows, 0, ds, 1, dC, n, 0);
  std::vector<double> C((size_t)n * n);
  cudaMemcpy(C.data(), dC, 8 * C.size(), cudaMemcpyDeviceToHost);
  double eg = 0;  // diag(1/s) U^T M = V^T
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) eg = fmax(eg, fabs(C[i + (size_t)j * n] - V[j + (size_t)i * n]));
  printf("gemm err %.3e\n", eg);
  return 0;
}
