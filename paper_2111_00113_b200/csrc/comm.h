// comm.h -- single-process loopback transport (comm.cu): P ranks in one process on one device.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

namespace sks {
constexpr int LOOP_MAXR = 16;
struct LoopGroup;
LoopGroup* loop_group_create(int n);
void loop_group_destroy(LoopGroup* g);
int loop_group_size(const LoopGroup* g);
cudaError_t loop_rank_init(LoopGroup* g, int rank);
void loop_rank_fini(LoopGroup* g, int rank);
cudaError_t loop_allreduce(LoopGroup* g, int r, double* buf, size_t cnt, cudaStream_t st);
cudaError_t loop_halo(LoopGroup* g, int r, double* vec, int64_t off, int64_t nz, int64_t plane, int G,
                      cudaStream_t st);
cudaError_t loop_allgather(LoopGroup* g, int r, const double* w, double* dst, int64_t maxn, cudaStream_t st);
}  // namespace sks
