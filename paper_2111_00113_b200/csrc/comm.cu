// comm.cu -- the single-process LOOPBACK transport: P ranks of libsks in one process (one host thread per rank,
// all on one device) exchanging halos, all-reductions and all-gathers with device-to-device copies ordered by
// CUDA events and host barriers, instead of NCCL.  It runs the library's own multi-rank code (row partition,
// ghost planes, per-rank partial sums, replicated small side) for P = 2, 4, ... when fewer GPUs than ranks exist.
//
// Semantics follow NCCL's stream semantics: every rank calls the same collectives in the same order on its main
// stream; each collective is (1) record `ready` after this rank's inputs on its stream, host barrier, every rank's
// stream waits for all `ready` events; (2) the data movement / fixed-order sum on this rank's stream; (3) record
// `done`, host barrier, every stream waits for all `done` events (no rank overwrites a buffer a peer still reads).
// No kernel ever waits on another rank's kernel: ordering is by stream-event dependencies only (B200_PROFILING:
// "do not run kernels that wait on one another ... on one GPU").  The all-reduce sums the ranks' contributions
// in rank order, so it is deterministic.  One cudaMemcpyAsync per copy (no batched copies).
#include <condition_variable>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "comm.h"

namespace sks {

struct LoopGroup {
  int n = 0;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<const void*> ptr;     // published per collective
  std::vector<int64_t> val;         // published per collective (e.g. a peer's plane count)
  std::vector<cudaEvent_t> ready, done;
  std::vector<double*> stage;       // all-reduce staging, one per rank (owned by that rank)
  std::vector<size_t> stage_cnt;
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const uint64_t g = gen;
    if (++arrived == n) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

LoopGroup* loop_group_create(int n) {
  if (n < 1 || n > LOOP_MAXR) return nullptr;
  LoopGroup* g = new LoopGroup();
  g->n = n;
  g->ptr.assign(n, nullptr);
  g->val.assign(n, 0);
  g->ready.assign(n, nullptr);
  g->done.assign(n, nullptr);
  g->stage.assign(n, nullptr);
  g->stage_cnt.assign(n, 0);
  return g;
}

void loop_group_destroy(LoopGroup* g) { delete g; }

int loop_group_size(const LoopGroup* g) { return g->n; }

cudaError_t loop_rank_init(LoopGroup* g, int rank) {
  cudaError_t e = cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&g->done[rank], cudaEventDisableTiming);
  return e;
}

void loop_rank_fini(LoopGroup* g, int rank) {
  if (g->ready[rank]) cudaEventDestroy(g->ready[rank]);
  if (g->done[rank]) cudaEventDestroy(g->done[rank]);
  if (g->stage[rank]) cudaFree(g->stage[rank]);
  g->ready[rank] = g->done[rank] = nullptr;
  g->stage[rank] = nullptr;
}

// phase 1: publish (p, v), record ready, barrier, wait for every rank's ready
static cudaError_t enter(LoopGroup* g, int r, const void* p, int64_t v, cudaStream_t st) {
  g->ptr[r] = p;
  g->val[r] = v;
  cudaError_t e = cudaEventRecord(g->ready[r], st);
  g->barrier();
  for (int q = 0; q < g->n && e == cudaSuccess; ++q)
    if (q != r) e = cudaStreamWaitEvent(st, g->ready[q], 0);
  return e;
}

// phase 3: record done, barrier, wait for every rank's done
static cudaError_t leave(LoopGroup* g, int r, cudaStream_t st) {
  cudaError_t e = cudaEventRecord(g->done[r], st);
  g->barrier();
  for (int q = 0; q < g->n && e == cudaSuccess; ++q)
    if (q != r) e = cudaStreamWaitEvent(st, g->done[q], 0);
  return e;
}

struct SumPtrs {
  const double* p[LOOP_MAXR];
};

__global__ void loop_sum_kernel(SumPtrs s, int n, size_t cnt, double* __restrict__ out) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < cnt; i += (size_t)gridDim.x * blockDim.x) {
    double t = s.p[0][i];
    for (int q = 1; q < n; ++q) t += s.p[q][i];  // rank order: deterministic
    out[i] = t;
  }
}

cudaError_t loop_allreduce(LoopGroup* g, int r, double* buf, size_t cnt, cudaStream_t st) {
  if (cnt == 0) return cudaSuccess;
  cudaError_t e = cudaSuccess;
  if (g->stage_cnt[r] < cnt) {  // grown only by its owner, never while a peer reads it (leave() of the last call)
    if (g->stage[r]) e = cudaFree(g->stage[r]);
    g->stage[r] = nullptr;
    if (e == cudaSuccess) e = cudaMalloc(&g->stage[r], sizeof(double) * cnt);
    if (e != cudaSuccess) return e;
    g->stage_cnt[r] = cnt;
  }
  e = cudaMemcpyAsync(g->stage[r], buf, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  if ((e = enter(g, r, g->stage[r], (int64_t)cnt, st)) != cudaSuccess) return e;
  SumPtrs sp;
  for (int q = 0; q < LOOP_MAXR; ++q) sp.p[q] = q < g->n ? static_cast<const double*>(g->ptr[q]) : nullptr;
  const int grid = (int)std::min<size_t>((cnt + 255) / 256, 1024);
  loop_sum_kernel<<<grid, 256, 0, st>>>(sp, g->n, cnt, buf);
  if ((e = cudaGetLastError()) != cudaSuccess) return e;
  return leave(g, r, st);
}

// ghost planes of vec (layout: G ghost planes, nz interior planes, G ghost planes of `plane` points): the low
// ghosts receive the last G interior planes of rank r-1, the high ghosts the first G interior planes of r+1
cudaError_t loop_halo(LoopGroup* g, int r, double* vec, int64_t off, int64_t nz, int64_t plane, int G,
                      cudaStream_t st) {
  cudaError_t e = enter(g, r, vec, nz, st);
  if (e != cudaSuccess) return e;
  const size_t cnt = (size_t)G * plane;
  if (r > 0) {
    const double* pv = static_cast<const double*>(g->ptr[r - 1]);
    const int64_t pnz = g->val[r - 1];
    e = cudaMemcpyAsync(vec + off - cnt, pv + off + (pnz - G) * plane, sizeof(double) * cnt,
                        cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  if (r + 1 < g->n) {
    const double* pv = static_cast<const double*>(g->ptr[r + 1]);
    e = cudaMemcpyAsync(vec + off + nz * plane, pv + off, sizeof(double) * cnt, cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) return e;
  }
  return leave(g, r, st);
}

// dst[q * maxn + i] = w_q[i], i < maxn, for every rank q (the CSR gathered-vector layout)
cudaError_t loop_allgather(LoopGroup* g, int r, const double* w, double* dst, int64_t maxn, cudaStream_t st) {
  cudaError_t e = enter(g, r, w, maxn, st);
  if (e != cudaSuccess) return e;
  for (int q = 0; q < g->n && e == cudaSuccess; ++q)
    e = cudaMemcpyAsync(dst + (int64_t)q * maxn, g->ptr[q], sizeof(double) * maxn, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) return e;
  return leave(g, r, st);
}

}  // namespace sks
