// Debug harness for hqr_kernel: reads n and an n x n column-major Hessenberg matrix (binary doubles),
// runs the kernel (optionally stopped after HQ_DEBUG_SWEEPS sweeps), writes H, wr, wi, info.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../../paper_2111_00113_b200/csrc/eig.cu"
int main(int argc, char** argv) {
  FILE* f = fopen(argv[1], "rb");
  int n;
  if (fread(&n, 4, 1, f) != 1) return 1;
  std::vector<double> h((size_t)n * n);
  if (fread(h.data(), 8, h.size(), f) != h.size()) return 1;
  fclose(f);
  double *dh, *wr, *wi;
  int* info;
  cudaMalloc(&dh, 8 * h.size());
  cudaMalloc(&wr, 8 * n);
  cudaMalloc(&wi, 8 * n);
  cudaMalloc(&info, 64);
  cudaMemset(info, 0, 64);
  const int K = argc > 3 ? atoi(argv[3]) : 0;
  cudaMemcpy(info + 7, &K, 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dh, h.data(), 8 * h.size(), cudaMemcpyHostToDevice);
  sks::launch_hqr(dh, n, n, wr, wi, info, 0);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> o(h.size() + 2 * n);
  int inf[8];
  cudaMemcpy(o.data(), dh, 8 * h.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data() + h.size(), wr, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(o.data() + h.size() + n, wi, 8 * n, cudaMemcpyDeviceToHost);
  cudaMemcpy(inf, info, 32, cudaMemcpyDeviceToHost);
  FILE* g = fopen(argv[2], "wb");
  fwrite(inf, 4, 8, g);
  fwrite(o.data(), 8, o.size(), g);
  fclose(g);
  printf("cuda: %s info %d sweeps %d steps %d\n", cudaGetErrorString(e), inf[0], inf[1], inf[2]);
  return 0;
}
