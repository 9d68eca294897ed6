// api.cu -- C-ABI (include/sks.h) and the host drivers of sGMRES / sRR.
//
// Driver structure:
//   main stream : residual/start kernel, one fused step kernel per basis column (stencil)
//                 or SpMV+orth (CSR), assembly; NCCL halo + partial-sum allreduce per column
//                 when nranks > 1.
//   side stream : every batch of up to 32 finished columns -> sketch batch (S W), then the
//                 incremental sketched QR of the reduced matrix (BCGS2 + panel) with r_est,j
//                 and the early-exit test.  Forks from / joins into the main stream.
//   host        : enqueues ahead, polls the early-exit flag of batch b-1 before enqueuing
//                 batch b+1 (bounded lag); one synchronisation per restart cycle.
#include <cuda_runtime.h>
#include <nccl.h>

#include <climits>
#include <map>
#include <mutex>
#include <utility>
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/sks.h"

// power-iteration steps of the kappa_2(T_j) estimate behind adaptive restarting
#define SKS_ADAPT_ITERS 16
#include "comm.h"
#include "common.cuh"
#include "internal.h"
#include "step.cuh"

using namespace sks;

namespace sks {
cudaError_t set_smem_attr_raw(const void* fn, size_t smem) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  size_t& cur = done[{fn, dev}];
  if (cur >= smem) return cudaSuccess;
  e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return e;
  }
  cur = smem;
  return cudaSuccess;
}
}  // namespace sks

// ------------------------------------------------------------------------------------
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct sks_ctx {
  int device = 0, rank = 0, nranks = 1, num_sms = 148;
  int main_sms = 146;  // SMs the persistent basis/sketch kernels use; the rest run the side stream's QR
  cudaStream_t own_main = nullptr, side = nullptr, user_main = nullptr;
  cudaStream_t aux = nullptr;  // per-cycle kappa(T) diagnostics on a copy of T, off the side stream's queue
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_t0 = nullptr, ev_t1 = nullptr, ev_b0 = nullptr,
              ev_b1 = nullptr, ev_aux = nullptr, ev_aux_done = nullptr;
  std::vector<cudaEvent_t> ev_batch;
  std::vector<cudaEvent_t> ev_step;  // SKS_OPT_TIME_STEPS: [2 i] before / [2 i + 1] after step launch i
  ncclComm_t comm = nullptr;
  LoopGroup* loop = nullptr;   // single-process loopback transport (comm.cu) instead of NCCL
  int ghost_min = 2;           // ghost planes per side of the next basis (matrix-powers Chebyshev: S + 1)
  std::string err = "";
  int64_t launches = 0;
  // workspaces
  DevBuf W, xb, fb, vb, mr, xg, part, part2, partsk, sigma, H, mnorm, SW, Xp, Zb, U, T, rvec, rho, rest, coef,
      ctrl, small, Mh, Mh2, wr, wi, sel, th, yr, yi, ework, SAB, SB, svw, svs, svU, svV, svH, y2r, y2i, Xr, Xi, AXr, AXi, rpb, cib, vab, cig, rbd,
      tmp, bgsw, bgsc, plan, gam, rcoef, srft_q, srft_w, partc, partcs, wz, wn, wpart, gsave, csync, cctrl, Tcopy, ellc, ellv;
  CtrlBlock* h_ctrl = nullptr;   // pinned mirror
  double* h_small = nullptr;     // pinned scratch (4096 doubles)
  int64_t w_zeroed_bytes = 0;
  void* tma_cache = nullptr;   // encoded tensor maps of the stencil step
  void* zm_cache = nullptr;    // encoded tensor maps of the 3D z-march step
  void* ym_cache = nullptr;    // encoded tensor maps of the 2D y-march step
  void* srft_cache = nullptr;  // cuFFT plans of the SRFT sketch
  int sketch_kind = 0;         // SKS_SKETCH_* of the running call
  uint64_t sk_seed = 0;        // its seed and current cycle (SRFT key)
  uint32_t sk_cycle = 0;
  int use_tma = 1;             // SKS_NO_TMA=1 forces the generic stencil kernels
  int tma_mask = 7;
  cudaStream_t main() const { return user_main ? user_main : own_main; }
};

static thread_local char g_err[512];

#define SKS_CK(ctx, expr)                                                                 \
  do {                                                                                   \
    cudaError_t _e = (expr);                                                             \
    if (_e != cudaSuccess) {                                                             \
      cudaGetLastError(); /* do not leak a non-sticky error into the next call */        \
      (ctx)->err = std::string(#expr) + ": " + cudaGetErrorString(_e);                  \
      return SKS_ECUDA;                                                                  \
    }                                                                                    \
  } while (0)

#define SKS_NC(ctx, expr)                                                                 \
  do {                                                                                   \
    ncclResult_t _r = (expr);                                                            \
    if (_r != ncclSuccess) {                                                             \
      (ctx)->err = std::string(#expr) + ": " + ncclGetErrorString(_r);                  \
      return SKS_ENCCL;                                                                  \
    }                                                                                    \
  } while (0)

#define SKS_TRY(expr)          \
  do {                         \
    sks_status _s = (expr);    \
    if (_s != SKS_OK) return _s; \
  } while (0)

static sks_status fail(sks_ctx* c, sks_status s, const std::string& m) {
  if (c) c->err = m;
  return s;
}

static sks_status ensure(sks_ctx* c, DevBuf& b, size_t bytes, bool zero = false) {
  if (bytes == 0) bytes = 8;
  if (b.bytes >= bytes) return SKS_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.bytes = 0;
  cudaError_t e = cudaMalloc(&b.p, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(c, SKS_ENOMEM, std::string("cudaMalloc(") + std::to_string(bytes) + "): " + cudaGetErrorString(e));
  }
  b.bytes = bytes;
  if (zero) SKS_CK(c, cudaMemsetAsync(b.p, 0, bytes, c->main()));
  return SKS_OK;
}

// ------------------------------------------------------------------------------------
// geometry of this rank's row block
struct Geo {
  int kind = 0, dim = 0;
  int64_t m = 0, n_global = 0, row_begin = 0, row_end = 0, n = 0;
  int64_t plane = 1, nz = 0, z0 = 0, G = 0, ld = 0, off = 0;
  double cc = 0, cm = 0, cp = 0;
};

static sks_status make_geo(sks_ctx* c, const sks_operator* A, Geo* g) {
  if (!A) return fail(c, SKS_EINVAL, "operator is NULL");
  g->kind = A->kind;
  g->n_global = A->n_global;
  g->row_begin = A->row_begin;
  g->row_end = A->row_end;
  g->n = A->row_end - A->row_begin;
  if (g->n <= 0 || A->row_begin < 0 || A->row_end > A->n_global)
    return fail(c, SKS_EINVAL, "bad row block [row_begin,row_end)");
  if (A->kind == SKS_OP_STENCIL2D || A->kind == SKS_OP_STENCIL3D) {
    g->dim = A->kind == SKS_OP_STENCIL2D ? 2 : 3;
    g->m = A->m;
    if (g->m < 2) return fail(c, SKS_EINVAL, "stencil m must be >= 2");
    g->plane = g->dim == 2 ? g->m : g->m * g->m;
    const int64_t ng = g->dim == 2 ? g->m * g->m : g->m * g->m * g->m;
    if (ng != A->n_global) return fail(c, SKS_EINVAL, "n_global != m^dim");
    if (A->row_begin % g->plane || A->row_end % g->plane)
      return fail(c, SKS_EINVAL, "stencil row block must consist of whole lines (2D) / planes (3D)");
    g->nz = g->n / g->plane;
    g->z0 = A->row_begin / g->plane;
    g->G = (std::max(2, c->ghost_min) + 1) & ~1;  // even: the interior offset G*plane stays 16-byte aligned
    if (c->nranks > 1 && g->nz < g->G) return fail(c, SKS_EINVAL, "each rank needs >= G planes/lines");
    if (!std::isfinite(A->beta)) return fail(c, SKS_EINVAL, "beta not finite");
    const double ih2 = (double)(g->m + 1) * (double)(g->m + 1);
    const double ih = (double)(g->m + 1) / 2.0;
    g->cc = 2.0 * g->dim * ih2;
    g->cm = -ih2 - A->beta * ih;
    g->cp = -ih2 + A->beta * ih;
    g->off = g->G * g->plane;
    g->ld = ((g->nz + 2 * g->G) * g->plane + 63) / 64 * 64;
  } else if (A->kind == SKS_OP_CSR) {
    g->dim = 0;
    g->plane = 1;
    g->nz = g->n;
    g->z0 = A->row_begin;
    g->G = 0;
    g->off = 0;
    g->ld = (g->n + 63) / 64 * 64;
    if (!A->row_ptr || !A->col_idx || !A->val) return fail(c, SKS_EINVAL, "CSR arrays are NULL");
  } else {
    return fail(c, SKS_EINVAL, "unknown operator kind");
  }
  if (A->n_global > INT_MAX && A->kind == SKS_OP_CSR)
    return fail(c, SKS_EUNSUPPORTED, "CSR with n_global >= 2^31 (int32 indices)");
  return SKS_OK;
}

// ------------------------------------------------------------------------------------
// communication (nranks > 1): halo planes of a ghost-layout vector, allreduce of partials
static sks_status halo_exchange(sks_ctx* c, const Geo& g, double* vec) {
  if (c->nranks == 1 || g.G == 0) return SKS_OK;
  if (c->loop) {
    SKS_CK(c, loop_halo(c->loop, c->rank, vec, g.off, g.nz, g.plane, (int)g.G, c->main()));
    return SKS_OK;
  }
  const size_t cnt = (size_t)(g.G * g.plane);
  const int lo = c->rank - 1, hi = c->rank + 1;
  SKS_NC(c, ncclGroupStart());
  if (lo >= 0) {
    SKS_NC(c, ncclSend(vec + g.off, cnt, ncclDouble, lo, c->comm, c->main()));
    SKS_NC(c, ncclRecv(vec + g.off - cnt, cnt, ncclDouble, lo, c->comm, c->main()));
  }
  if (hi < c->nranks) {
    SKS_NC(c, ncclSend(vec + g.off + (g.nz - g.G) * g.plane, cnt, ncclDouble, hi, c->comm, c->main()));
    SKS_NC(c, ncclRecv(vec + g.off + g.nz * g.plane, cnt, ncclDouble, hi, c->comm, c->main()));
  }
  SKS_NC(c, ncclGroupEnd());
  return SKS_OK;
}

static sks_status allreduce_sum(sks_ctx* c, double* buf, size_t cnt, cudaStream_t st) {
  if (c->nranks == 1) return SKS_OK;
  if (c->loop) {
    SKS_CK(c, loop_allreduce(c->loop, c->rank, buf, cnt, st));
    return SKS_OK;
  }
  SKS_NC(c, ncclAllReduce(buf, buf, cnt, ncclDouble, ncclSum, c->comm, st));
  return SKS_OK;
}

// Per-CTA partial sums [grid][SKS_NP] of a step launch at nranks > 1: reduced on the device, in a
// fixed order, into row 0 (in place: thread i reads only component i), then the SKS_NP scalars
// (k + 3 dots and norms, 88 bytes) are all-reduced.  The consumer then reads grid_prev = 1 row, so
// ranks whose step grids differ (uneven slabs) never see stale rows of the ping-pong slot.
static sks_status reduce_partials(sks_ctx* c, double* slot, int grid, cudaStream_t st) {
  if (c->nranks == 1) return SKS_OK;
  SKS_CK(c, launch_sum_partials(slot, grid, SKS_NP, SKS_NP, slot, st));
  ++c->launches;
  return allreduce_sum(c, slot, SKS_NP, st);
}

// CSR: make w (n_local rows) available as the gathered vector for the SpMV
static sks_status csr_gather(sks_ctx* c, const Geo& g, const double* w, const double** xg, int64_t maxn) {
  if (c->nranks == 1) {
    *xg = w;
    return SKS_OK;
  }
  double* dst = c->xg.as<double>();
  if (c->loop) {
    SKS_CK(c, loop_allgather(c->loop, c->rank, w, dst, maxn, c->main()));
    *xg = dst;
    return SKS_OK;
  }
  SKS_NC(c, ncclAllGather(w, dst, (size_t)maxn, ncclDouble, c->comm, c->main()));
  *xg = dst;
  return SKS_OK;
}

// ------------------------------------------------------------------------------------
extern "C" {

int sks_abi_version(void) { return SKS_ABI_VERSION; }

const char* sks_last_error(const sks_ctx* ctx) {
  if (!ctx) return g_err;
  return ctx->err.c_str();
}

sks_status sks_get_unique_id(unsigned char id[128]) {
  if (!id) return SKS_EINVAL;
  ncclUniqueId u;
  ncclResult_t r = ncclGetUniqueId(&u);
  if (r != ncclSuccess) {
    snprintf(g_err, sizeof(g_err), "ncclGetUniqueId: %s", ncclGetErrorString(r));
    return SKS_ENCCL;
  }
  static_assert(sizeof(u.internal) == 128, "nccl id size");
  memcpy(id, u.internal, 128);
  return SKS_OK;
}

sks_status sks_partition(int kind, int64_t m, int64_t n_global, int nranks, int rank, int64_t* row_begin,
                         int64_t* row_end) {
  if (!row_begin || !row_end || nranks < 1 || rank < 0 || rank >= nranks) return SKS_EINVAL;
  int64_t unit, count;
  if (kind == SKS_OP_CSR) {
    unit = 1;
    count = n_global;
  } else if (kind == SKS_OP_STENCIL2D) {
    unit = m;
    count = m;
  } else if (kind == SKS_OP_STENCIL3D) {
    unit = m * m;
    count = m;
  } else {
    return SKS_EINVAL;
  }
  const int64_t base = count / nranks, rem = count % nranks;
  const int64_t lo = rank * base + std::min<int64_t>(rank, rem);
  const int64_t hi = lo + base + (rank < rem ? 1 : 0);
  *row_begin = lo * unit;
  *row_end = hi * unit;
  return SKS_OK;
}

static sks_status create_ctx(sks_ctx** out, int device, int rank, int nranks, const unsigned char* id,
                             LoopGroup* loop);

sks_status sks_create(sks_ctx** out, int device, int rank, int nranks, const unsigned char* id) {
  return create_ctx(out, device, rank, nranks, id, nullptr);
}

sks_status sks_loopback_create(int nranks, sks_loopback** group) {
  if (!group || nranks < 1 || nranks > LOOP_MAXR) return SKS_EINVAL;
  *group = reinterpret_cast<sks_loopback*>(loop_group_create(nranks));
  return *group ? SKS_OK : SKS_ENOMEM;
}

sks_status sks_loopback_destroy(sks_loopback* group) {
  if (group) loop_group_destroy(reinterpret_cast<LoopGroup*>(group));
  return SKS_OK;
}

sks_status sks_create_loopback(sks_ctx** out, int device, int rank, sks_loopback* group) {
  if (!group) return SKS_EINVAL;
  LoopGroup* g = reinterpret_cast<LoopGroup*>(group);
  return create_ctx(out, device, rank, loop_group_size(g), nullptr, g);
}

static sks_status create_ctx(sks_ctx** out, int device, int rank, int nranks, const unsigned char* id,
                             LoopGroup* loop) {
  if (!out) return SKS_EINVAL;
  *out = nullptr;
  if (nranks < 1 || rank < 0 || rank >= nranks) return SKS_EINVAL;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    snprintf(g_err, sizeof(g_err), "no CUDA device available (%s); libsks has no CPU fallback",
             e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
    return SKS_ECUDA;
  }
  if (device < 0 || device >= ndev) {
    snprintf(g_err, sizeof(g_err), "device %d out of range (%d devices)", device, ndev);
    return SKS_EINVAL;
  }
  sks_ctx* c = new sks_ctx();
  c->device = device;
  {
    const char* e = getenv("SKS_NO_TMA");
    c->use_tma = !(e && e[0] == '1');
    const char* mk = getenv("SKS_TMA_MASK");  // debug: bit i = use TMA for step mode i
    c->tma_mask = mk ? atoi(mk) : 7;
  }
  c->rank = rank;
  c->nranks = nranks;
  cudaSetDevice(device);
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  {
    const char* e = getenv("SKS_RESERVE_SMS");  // SMs kept free for the side stream (default 2)
    const int r = e ? atoi(e) : 2;
    c->main_sms = std::max(1, c->num_sms - std::max(0, r));
  }
  cudaStreamCreateWithFlags(&c->own_main, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&c->ev_aux, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_aux_done, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming);
  cudaEventCreate(&c->ev_t0);
  cudaEventCreate(&c->ev_t1);
  cudaEventCreate(&c->ev_b0);
  cudaEventCreate(&c->ev_b1);
  c->ev_batch.resize(256);
  for (auto& ev : c->ev_batch) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (cudaMallocHost(&c->h_ctrl, sizeof(CtrlBlock)) != cudaSuccess ||
      cudaMallocHost(&c->h_small, 4096 * sizeof(double)) != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "cudaMallocHost failed");
    delete c;
    return SKS_ENOMEM;
  }
  if (loop) {
    c->loop = loop;
    if (loop_rank_init(loop, rank) != cudaSuccess) {
      snprintf(g_err, sizeof(g_err), "loopback rank init failed");
      delete c;
      return SKS_ECUDA;
    }
  } else if (nranks > 1) {
    if (!id) {
      snprintf(g_err, sizeof(g_err), "nranks > 1 needs the NCCL unique id");
      delete c;
      return SKS_EINVAL;
    }
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, u, rank);
    if (r != ncclSuccess) {
      snprintf(g_err, sizeof(g_err), "ncclCommInitRank: %s", ncclGetErrorString(r));
      delete c;
      return SKS_ENCCL;
    }
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof(g_err), "context setup: %s", cudaGetErrorString(e));
    delete c;
    return SKS_ECUDA;
  }
  *out = c;
  return SKS_OK;
}

sks_status sks_destroy(sks_ctx* c) {
  if (!c) return SKS_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  DevBuf* bufs[] = {&c->W,    &c->xb,   &c->fb,    &c->vb,   &c->mr,   &c->xg,   &c->part,  &c->part2, &c->partsk,
                    &c->sigma, &c->H,   &c->mnorm, &c->SW,   &c->Xp,   &c->Zb,   &c->U,     &c->T,     &c->rvec,
                    &c->rho,  &c->rest, &c->coef,  &c->ctrl, &c->small, &c->Mh,  &c->Mh2,   &c->wr,    &c->wi,
                    &c->sel,  &c->th,   &c->yr,    &c->yi,   &c->ework, &c->SAB, &c->SB,    &c->Xr,    &c->Xi,
                    &c->AXr,  &c->AXi,  &c->rpb,   &c->cib,  &c->vab,  &c->cig,  &c->rbd,   &c->tmp,
                    &c->bgsw, &c->bgsc, &c->plan, &c->gam, &c->rcoef, &c->srft_q, &c->srft_w, &c->partc, &c->partcs, &c->wz, &c->wn, &c->wpart, &c->gsave, &c->csync, &c->cctrl, &c->Tcopy,
                    &c->svw,  &c->svs,  &c->svU,   &c->svV,  &c->svH,  &c->y2r,   &c->y2i};
  for (DevBuf* b : bufs)
    if (b->p) cudaFree(b->p);
  if (c->comm) ncclCommDestroy(c->comm);
  if (c->loop) loop_rank_fini(c->loop, c->rank);
  if (c->tma_cache) stencil_tma_free(c->tma_cache);
  if (c->zm_cache) stencil_zm_free(c->zm_cache);
  if (c->ym_cache) stencil_ym_free(c->ym_cache);
  if (c->srft_cache) srft_free(c->srft_cache);
  for (auto& ev : c->ev_batch) cudaEventDestroy(ev);
  for (auto& ev : c->ev_step) cudaEventDestroy(ev);
  cudaEvent_t evs[] = {c->ev_fork, c->ev_join, c->ev_t0, c->ev_t1, c->ev_b0, c->ev_b1, c->ev_aux, c->ev_aux_done};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  if (c->own_main) cudaStreamDestroy(c->own_main);
  if (c->side) cudaStreamDestroy(c->side);
  if (c->aux) cudaStreamDestroy(c->aux);
  if (c->h_ctrl) cudaFreeHost(c->h_ctrl);
  if (c->h_small) cudaFreeHost(c->h_small);
  delete c;
  return SKS_OK;
}

sks_status sks_set_stream(sks_ctx* c, void* stream) {
  if (!c) return SKS_EINVAL;
  c->user_main = reinterpret_cast<cudaStream_t>(stream);
  return SKS_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------------------
// shared helpers of the drivers
// ------------------------------------------------------------------------------------
namespace {

struct Basis {
  sks_ctx* c;
  Geo g;
  int k;
  int ncol;            // columns allocated
  int ldH;
  int step_grid = 0;   // stencil step grid, or CSR grid
  bool tma = false;    // TMA-fed stencil kernels
  bool zm = false;     // 3D z-march kernel (replaces the TMA box kernel)
  bool ym = false;     // 2D y-march kernel (replaces the TMA box kernel)
  int last_grid = 0;   // grid of the previous step launch (its partial count)
  StepArgs sat;        // step arguments with the TMA tiling
  int tma_grid = 0;
  int pslots = 0;      // partial slots (fixed across ranks)
  bool defer = false;  // deferred Chebyshev bookkeeping (StepArgs::defer)
  int mpk_s = 0;       // 2D Chebyshev matrix-powers steps: columns per launch (0 = off)
  int mpk_grid = 0;
  bool coop = false;   // small single-rank stencil problem: batches of columns in one cooperative launch
  int coop_grid = 0;
  int coop1_lines = 0; // > 0: the one-barrier-per-column 2D kernel (step_coop1_kernel), lines per CTA
  int fin_next = 2;    // first column whose deferred bookkeeping is pending
  int defer_grid = 0;  // step grid of the deferred launches (per-column partial rows)
  StepArgs sa;
  // CSR
  const int32_t* rp = nullptr;
  const int32_t* ci = nullptr;
  const double* va = nullptr;
  const int32_t* ell_ci = nullptr;  // ELL copy (column-major [ell_w][n]) when the rows are near-uniform
  const double* ell_va = nullptr;
  int ell_w = 0;
  int64_t maxn = 0;    // max local rows over ranks (CSR gather)
  int64_t nnz = 0;
  double bytes = 0.0;  // algorithmic bytes of the basis loop
  int64_t steps = 0;
  bool time_steps = false;  // bracket step launches with events (SKS_OPT_TIME_STEPS)
  int time_stride = 1;      // ... every time_stride-th launch
  int time_window = 1;      // > 1: one event pair around time_window consecutive step launches inside a sketch batch
                            // (keeps the programmatic overlap between the window's launches; SKS_TIME_WINDOW)
  int win_end = -1;         // last column of the open window, -1 = none
  double win_bytes = 0.0;
  int64_t launches_timed = 0;  // step launches covered by the recorded event pairs
  int ntimed = 0;           // event pairs recorded in this cycle
  double bytes_timed = 0.0; // algorithmic bytes of the timed launches (this cycle)
};

static double* colp(sks_ctx* c, const Basis& b, int j) { return c->W.as<double>() + (int64_t)j * b.g.ld; }

static sks_status setup_basis(sks_ctx* c, const sks_operator* A, int k, int ncol, Basis* b) {
  b->c = c;
  SKS_TRY(make_geo(c, A, &b->g));
  b->k = k;
  b->ncol = ncol;
  b->ldH = ncol + 1;
  const Geo& g = b->g;
  const size_t wbytes = sizeof(double) * (size_t)g.ld * ncol;
  const bool fresh_w = c->W.bytes < wbytes;
  SKS_TRY(ensure(c, c->W, wbytes));
  (void)fresh_w;
  if (g.G > 0) {
    // ghost planes must be zero at the physical boundary (Dirichlet) for THIS geometry:
    // clear the G leading and G trailing planes (+ pitch padding) of every column.
    const size_t head = sizeof(double) * (size_t)(g.G * g.plane);
    const size_t tail_off = sizeof(double) * (size_t)(g.off + g.nz * g.plane);
    const size_t tail = sizeof(double) * (size_t)g.ld - tail_off;
    SKS_CK(c, cudaMemset2DAsync(c->W.p, sizeof(double) * g.ld, 0, head, ncol, c->main()));
    SKS_CK(c, cudaMemset2DAsync(c->W.as<char>() + tail_off, sizeof(double) * g.ld, 0, tail, ncol, c->main()));
  }
  SKS_TRY(ensure(c, c->xb, sizeof(double) * g.ld));
  SKS_TRY(ensure(c, c->fb, sizeof(double) * g.ld));
  SKS_TRY(ensure(c, c->vb, sizeof(double) * g.ld));
  SKS_TRY(ensure(c, c->sigma, sizeof(double) * (ncol + 2), true));
  SKS_TRY(ensure(c, c->H, sizeof(double) * (size_t)(ncol + 1) * (ncol + 1)));
  SKS_CK(c, cudaMemsetAsync(c->H.p, 0, sizeof(double) * (size_t)(ncol + 1) * (ncol + 1), c->main()));
  SKS_TRY(ensure(c, c->mnorm, sizeof(double) * (ncol + 2), true));
  SKS_TRY(ensure(c, c->gam, sizeof(double) * (ncol + 2)));
  {
    std::vector<double> ones(ncol + 2, 1.0);  // gam_i = 1 unless a Chebyshev step sets it
    SKS_CK(c, cudaMemcpy(c->gam.p, ones.data(), sizeof(double) * (ncol + 2), cudaMemcpyHostToDevice));
  }
  SKS_TRY(ensure(c, c->ctrl, sizeof(CtrlBlock), true));
  SKS_TRY(ensure(c, c->small, sizeof(double) * 4096, true));
  b->pslots = c->num_sms * 4;
  SKS_TRY(ensure(c, c->part, sizeof(double) * (size_t)2 * b->pslots * SKS_NP));
  SKS_TRY(ensure(c, c->part2, sizeof(double) * (size_t)2 * b->pslots * SKS_NP));
  SKS_CK(c, cudaMemsetAsync(c->part.p, 0, c->part.bytes, c->main()));
  SKS_CK(c, cudaMemsetAsync(c->part2.p, 0, c->part2.bytes, c->main()));
  if (g.kind != SKS_OP_CSR) {
    StepArgs& a = b->sa;
    memset(&a, 0, sizeof(a));
    a.m = g.m;
    a.nz = g.nz;
    a.z0 = g.z0;
    a.plane = g.plane;
    a.ld = g.ld;
    a.off = g.off;
    a.G = (int)g.G;
    a.dim = g.dim;
    a.cc = g.cc;
    a.cm = g.cm;
    a.cp = g.cp;
    a.k = k;
    a.W = c->W.as<double>();
    a.sigma = c->sigma.as<double>();
    a.H = c->H.as<double>();
    a.ldH = b->ldH;
    a.mnorm = c->mnorm.as<double>();
    a.gam = c->gam.as<double>();
    a.basis = 0;
    a.ctrl = c->ctrl.as<CtrlBlock>();
    b->tma = c->use_tma && stencil_tma_supported(g.dim, g.m, k);
    b->sat = a;
    stencil_tiling(g.dim, g.m, g.nz, c->main_sms, &a, &b->step_grid);
    if (b->step_grid > b->pslots) b->step_grid = b->pslots;
    b->zm = c->use_tma && stencil_zm_supported(g.dim, g.m, k);
    b->ym = !b->zm && c->use_tma && stencil_ym_supported(g.dim, g.m, k);
    if (b->zm) {
      b->tma = true;
      stencil_zm_tiling(g.m, g.nz, c->main_sms, &b->sat, &b->tma_grid);
      if (b->tma_grid > b->pslots) b->tma_grid = b->pslots;
    } else if (b->ym) {
      b->tma = true;
      stencil_ym_tiling(g.m, g.nz, c->main_sms, &b->sat, &b->tma_grid);
      if (b->tma_grid > b->pslots) b->tma_grid = b->pslots;
    } else if (b->tma) {
      stencil_tma_tiling(g.dim, g.m, g.nz, c->main_sms, &b->sat, &b->tma_grid);
      if (b->tma_grid > b->pslots) b->tma_grid = b->pslots;
    }
    {  // SKS_COOP_MAXN=n: problems up to n rows run batches of columns as one cooperative launch (P = 1).
       // Measured slower at C2 (19.6 vs 14.5 us per column: two grid barriers per column), so off by default
       // (profiles/r02/coop_ab_r02.txt)
      int64_t lim = 0;
      if (const char* e = getenv("SKS_COOP_MAXN")) lim = atoll(e);
      if (c->nranks == 1 && g.n <= lim) {
        b->coop_grid = std::min(coop_grid(c->main_sms), b->pslots);
        b->coop = b->coop_grid > 0;
      }
      // SKS_COOP1_MAXN (2D, P = 1): one cooperative launch per batch with one grid barrier per column and a
      // recomputed halo line (step_coop1_kernel)
      int64_t lim1 = 0;
      if (const char* e = getenv("SKS_COOP1_MAXN")) lim1 = atoll(e);
      if (c->nranks == 1 && g.n <= lim1 && !b->coop) {
        b->coop1_lines = coop1_lines(g.dim, g.m, g.nz, b->k, std::min(c->main_sms, b->pslots));
        if (b->coop1_lines > 0) {
          b->coop = true;
          b->coop_grid = (int)((g.nz + b->coop1_lines - 1) / b->coop1_lines);
        }
      }
      if (b->coop) {
        SKS_TRY(ensure(c, c->csync, 512, true));  // counter, flag, reduced partials (stencil_coop.cu)
        SKS_TRY(ensure(c, c->cctrl, sizeof(CtrlBlock), true));
      }
    }
  } else {
    b->step_grid = c->num_sms * 4;
    b->nnz = A->nnz_local;
    // device copies of the CSR arrays
    SKS_TRY(ensure(c, c->rpb, sizeof(int32_t) * (g.n + 1)));
    SKS_TRY(ensure(c, c->cib, sizeof(int32_t) * std::max<int64_t>(b->nnz, 1)));
    SKS_TRY(ensure(c, c->vab, sizeof(double) * std::max<int64_t>(b->nnz, 1)));
    SKS_CK(c, cudaMemcpyAsync(c->rpb.p, A->row_ptr, sizeof(int32_t) * (g.n + 1), cudaMemcpyDefault, c->main()));
    SKS_CK(c, cudaMemcpyAsync(c->cib.p, A->col_idx, sizeof(int32_t) * b->nnz, cudaMemcpyDefault, c->main()));
    SKS_CK(c, cudaMemcpyAsync(c->vab.p, A->val, sizeof(double) * b->nnz, cudaMemcpyDefault, c->main()));
    SKS_TRY(ensure(c, c->mr, sizeof(double) * g.ld));
    b->rp = c->rpb.as<int32_t>();
    b->ci = c->cib.as<int32_t>();
    b->va = c->vab.as<double>();
    if (c->nranks > 1) {
      // gathered-vector layout [rank][maxn]; remap global column indices once
      std::vector<int64_t> rb(c->nranks + 1);
      for (int r = 0; r < c->nranks; ++r) {
        int64_t lo, hi;
        sks_partition(SKS_OP_CSR, 0, g.n_global, c->nranks, r, &lo, &hi);
        rb[r] = lo;
        b->maxn = std::max(b->maxn, hi - lo);
      }
      rb[c->nranks] = g.n_global;
      if (rb[c->rank] != g.row_begin) return fail(c, SKS_EINVAL, "CSR row block must follow sks_partition");
      SKS_TRY(ensure(c, c->rbd, sizeof(int64_t) * (c->nranks + 1)));
      SKS_CK(c, cudaMemcpyAsync(c->rbd.p, rb.data(), sizeof(int64_t) * (c->nranks + 1), cudaMemcpyHostToDevice,
                                c->main()));
      SKS_TRY(ensure(c, c->cig, sizeof(int32_t) * std::max<int64_t>(b->nnz, 1)));
      SKS_CK(c, launch_remap_cols(b->nnz, b->ci, c->cig.as<int32_t>(), c->nranks, c->rbd.as<int64_t>(), b->maxn,
                                  c->main()));
      b->ci = c->cig.as<int32_t>();
      SKS_TRY(ensure(c, c->xg, sizeof(double) * (size_t)b->maxn * c->nranks));
      // every column must be readable up to maxn rows for the all-gather
      if (b->maxn > g.ld) return fail(c, SKS_EINVAL, "internal: maxn > ld");
    }
    // ELL copy for the SpMV when the longest row is short and close to the average (C4: <= 17 per row):
    // SKS_CSR_ELL=0 keeps the CSR kernel
    {
      const char* e = getenv("SKS_CSR_ELL");
      const bool want = !(e && e[0] == '0');
      if (want && g.n > 0) {
        int* dmax = reinterpret_cast<int*>(c->small.p);
        SKS_CK(c, launch_csr_max_row(g.n, b->rp, dmax, c->main()));
        int wmax = 0;
        SKS_CK(c, cudaMemcpyAsync(&wmax, dmax, sizeof(int), cudaMemcpyDeviceToHost, c->main()));
        SKS_CK(c, cudaStreamSynchronize(c->main()));
        const double avg = (double)b->nnz / (double)g.n;
        if (wmax > 0 && wmax <= 32 && wmax <= 1.25 * avg + 1.0) {
          SKS_TRY(ensure(c, c->ellc, sizeof(int32_t) * (size_t)wmax * g.n));
          SKS_TRY(ensure(c, c->ellv, sizeof(double) * (size_t)wmax * g.n));
          SKS_CK(c, launch_csr_to_ell(g.n, b->rp, b->ci, b->va, wmax, c->ellc.as<int32_t>(), c->ellv.as<double>(),
                                      c->main()));
          b->ell_ci = c->ellc.as<int32_t>();
          b->ell_va = c->ellv.as<double>();
          b->ell_w = wmax;
        }
      }
    }
    SKS_CK(c, cudaStreamSynchronize(c->main()));  // host CSR arrays may be freed after return
  }
  SKS_CK(c, cudaMemsetAsync(c->part.p, 0, c->part.bytes, c->main()));
  return SKS_OK;
}

// Chebyshev basis (Eq. Chebrecurse): k = 2 internally (the recurrence reads w_{j-1}
// and w_{j-2}); the spectral box defaults to the closed form of the stencil operator:
// eigenvalues of the 1D factor a + 2 sqrt(bc) cos(p pi/(m+1)) (real if bc >= 0), summed over
// the dim axes (Kronecker sum).
static sks_status set_basis(sks_ctx* c, const sks_operator* A, Basis& b, int basis, double bc_, double bdx,
                            double bdy) {
  if (basis == SKS_BASIS_ARNOLDI) return SKS_OK;
  if (basis != SKS_BASIS_CHEBYSHEV) return fail(c, SKS_EINVAL, "unknown basis kind");
  if (b.g.kind == SKS_OP_CSR) return fail(c, SKS_EUNSUPPORTED, "Chebyshev basis needs a stencil operator");
  if (bdx == 0.0 && bdy == 0.0) {
    const double m1 = (double)(b.g.m + 1);
    const double ih2 = m1 * m1, ih = m1 / 2.0;
    const double a1 = 2.0 * ih2, b1 = -ih2 - A->beta * ih, c1 = -ih2 + A->beta * ih;
    const double cosm = std::cos(M_PI / m1);
    bc_ = b.g.dim * a1;
    if (b1 * c1 >= 0.0) {
      bdx = b.g.dim * 2.0 * std::sqrt(b1 * c1) * cosm;
      bdy = 0.0;
    } else {
      bdx = 0.0;
      bdy = b.g.dim * 2.0 * std::sqrt(-b1 * c1) * cosm;
    }
  }
  const double rho = std::max(bdx, bdy);
  if (!(rho > 0.0) || !std::isfinite(rho) || !std::isfinite(bc_)) return fail(c, SKS_EINVAL, "bad Chebyshev box");
  const char* sync = getenv("SKS_CHEB_SYNC");  // 1: per-column reduction as for Arnoldi (A/B)
  b.defer = !(sync && sync[0] == '1') && b.g.kind != SKS_OP_CSR && !b.coop;  // coop reduces in-kernel
  if (b.defer) {
    SKS_TRY(ensure(c, c->partc, sizeof(double) * (size_t)(b.ncol + 2) * b.pslots * SKS_NP));
    SKS_TRY(ensure(c, c->partcs, sizeof(double) * (size_t)(b.ncol + 2) * SKS_NP));
  }
  for (StepArgs* a : {&b.sa, &b.sat}) {
    a->defer = b.defer ? 1 : 0;
    a->basis = 1;
    a->k = 2;
    a->cheb_c = bc_;
    a->cheb_rho = rho;
    a->cheb_e = (bdx * bdx - bdy * bdy) / (4.0 * rho);
  }
  b.k = 2;
  return SKS_OK;
}

// partial-slot pointer (ping-pong)
static double* pslot(sks_ctx* c, const Basis& b, DevBuf& buf, int j) {
  return buf.as<double>() + (size_t)(j & 1) * b.pslots * SKS_NP;
}

// first column: mode 1 (w_0 = f - A x) or mode 2 (w_0 = v), into W[:,0]; partials in slot 0
static sks_status first_column(sks_ctx* c, Basis& b, int mode, const double* xvec, const double* fvec) {
  cudaStream_t st = c->main();
  const Geo& g = b.g;
  double* p0 = pslot(c, b, c->part, 0);
  if (g.kind != SKS_OP_CSR) {
    const bool use_t = b.tma && (c->tma_mask >> mode & 1);
    StepArgs a = use_t ? b.sat : b.sa;
    a.mode = mode;
    a.j = 0;
    a.xin = xvec;
    a.fin = fvec;
    a.partials_out = p0;
    a.partials_in = nullptr;
    a.grid_prev = 0;
    b.last_grid = use_t ? b.tma_grid : b.step_grid;
    if (use_t && b.zm)
      SKS_CK(c, launch_step_stencil_zm(a, c->W.as<double>(), b.ncol, c->xb.as<double>(), c->fb.as<double>(),
                                       c->vb.as<double>(), b.tma_grid, st, &c->zm_cache));
    else if (use_t && b.ym)
      SKS_CK(c, launch_step_stencil_ym(a, c->W.as<double>(), b.ncol, c->xb.as<double>(), c->fb.as<double>(),
                                       c->vb.as<double>(), b.tma_grid, st, &c->ym_cache));
    else if (use_t)
      SKS_CK(c, launch_step_stencil_tma(a, c->W.as<double>(), b.ncol, c->xb.as<double>(), c->fb.as<double>(),
                                        c->vb.as<double>(), b.tma_grid, st, &c->tma_cache));
    else
      SKS_CK(c, launch_step_stencil(a, b.step_grid, st));
    ++c->launches;
    b.bytes += 8.0 * g.n * (mode == 1 ? 3 : 2);
  } else {
    b.last_grid = b.step_grid;
    if (mode == 1) {
      const double* xg = nullptr;
      SKS_TRY(csr_gather(c, g, xvec, &xg, b.maxn));
      SKS_CK(c, launch_csr_spmv(g.n, b.rp, b.ci, b.va, xg, colp(c, b, 0), fvec, 1, nullptr, 0, 0, 0, b.k, p0,
                                b.step_grid, st, nullptr, b.ell_ci, b.ell_va, b.ell_w));
    } else {
      SKS_CK(c, launch_copy_norm(g.n, xvec, colp(c, b, 0), p0, b.step_grid, st));
    }
    ++c->launches;
    b.bytes += (mode == 1) ? 12.0 * b.nnz + 4.0 * (g.n + 1) + 8.0 * 3 * g.n : 16.0 * g.n;
  }
  SKS_TRY(reduce_partials(c, p0, b.last_grid, st));
  SKS_TRY(halo_exchange(c, g, colp(c, b, 0)));
  ++b.steps;
  return SKS_OK;
}

// produce column j >= 1
static sks_status step_column(sks_ctx* c, Basis& b, int j) {
  cudaStream_t st = c->main();
  const Geo& g = b.g;
  const int grid_prev = c->nranks > 1 ? 1 : b.step_grid;
  const int nwin = std::min(b.k, j);
  if (g.kind != SKS_OP_CSR) {
    const bool use_t = b.tma && (c->tma_mask & 1);
    StepArgs a = use_t ? b.sat : b.sa;
    a.mode = 0;
    a.j = j;
    const bool tm = b.time_steps && b.time_window <= 1 && j % b.time_stride == 0 &&
                    2 * b.ntimed + 1 < (int)c->ev_step.size();
    if (tm) SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed], st));
    a.partials_in = pslot(c, b, c->part, j - 1);
    a.grid_prev = c->nranks > 1 ? 1 : b.last_grid;
    const bool dcol = b.defer && j >= 2;  // this column's partials go to its own slot (cheb_finalize)
    a.partials_out = dcol ? c->partc.as<double>() + (size_t)j * b.pslots * SKS_NP : pslot(c, b, c->part, j);
    b.last_grid = use_t ? b.tma_grid : b.step_grid;
    if (dcol) b.defer_grid = b.last_grid;
    if (use_t && b.zm)
      SKS_CK(c, launch_step_stencil_zm(a, c->W.as<double>(), b.ncol, c->xb.as<double>(), c->fb.as<double>(),
                                       c->vb.as<double>(), b.tma_grid, st, &c->zm_cache));
    else if (use_t && b.ym)
      SKS_CK(c, launch_step_stencil_ym(a, c->W.as<double>(), b.ncol, c->xb.as<double>(), c->fb.as<double>(),
                                       c->vb.as<double>(), b.tma_grid, st, &c->ym_cache));
    else if (use_t)
      SKS_CK(c, launch_step_stencil_tma(a, c->W.as<double>(), b.ncol, c->xb.as<double>(), c->fb.as<double>(),
                                        c->vb.as<double>(), b.tma_grid, st, &c->tma_cache));
    else
      SKS_CK(c, launch_step_stencil(a, b.step_grid, st));
    ++c->launches;
    if (tm) {
      SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed + 1], st));
      ++b.ntimed;
      ++b.launches_timed;
      b.bytes_timed += 8.0 * g.n * (nwin + 1);
    }
    if (b.win_end >= 0) b.win_bytes += 8.0 * g.n * (nwin + 1);
    if (!dcol) SKS_TRY(reduce_partials(c, a.partials_out, b.last_grid, st));  // deferred: once per batch
    SKS_TRY(halo_exchange(c, g, colp(c, b, j)));
    b.bytes += 8.0 * g.n * (nwin + 1);
  } else {
    const int lo = std::max(0, j - b.k), nw = j - lo;
    const double* xg = nullptr;
    const bool tm = b.time_steps && j % b.time_stride == 0 && 2 * b.ntimed + 1 < (int)c->ev_step.size();
    if (tm) SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed], st));
    SKS_TRY(csr_gather(c, g, colp(c, b, j - 1), &xg, b.maxn));
    double* pd = c->part2.as<double>();  // spmv partials (single slot)
    SKS_CK(c, launch_csr_spmv(g.n, b.rp, b.ci, b.va, xg, c->mr.as<double>(), nullptr, 0, c->W.as<double>(), g.ld,
                              lo, nw, b.k, pd, b.step_grid, st, c->ctrl.as<CtrlBlock>(), b.ell_ci, b.ell_va,
                              b.ell_w));
    SKS_TRY(reduce_partials(c, pd, b.step_grid, st));
    SKS_CK(c, launch_csr_orth(g.n, j, b.k, c->W.as<double>(), g.ld, c->mr.as<double>(), pslot(c, b, c->part, j - 1),
                              grid_prev, pd, grid_prev, pslot(c, b, c->part, j), c->sigma.as<double>(),
                              c->H.as<double>(), b.ldH, c->mnorm.as<double>(), c->ctrl.as<CtrlBlock>(),
                              b.step_grid, st));
    SKS_TRY(reduce_partials(c, pslot(c, b, c->part, j), b.step_grid, st));
    c->launches += 2;
    if (tm) {
      SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed + 1], st));
      ++b.ntimed;
      ++b.launches_timed;
      b.bytes_timed += 12.0 * b.nnz + 4.0 * (g.n + 1) + 8.0 * g.n * (nwin + 1);
    }
    b.bytes += 12.0 * b.nnz + 4.0 * (g.n + 1) + 8.0 * g.n * (nwin + 1);
  }
  ++b.steps;
  return SKS_OK;
}

// columns j0..j1 in one cooperative launch (Basis::coop)
static sks_status coop_columns(sks_ctx* c, Basis& b, int j0, int j1) {
  cudaStream_t st = c->main();
  const Geo& g = b.g;
  StepArgs a = b.sa;
  a.defer = 0;
  a.ctrl = c->cctrl.as<CtrlBlock>();
  SKS_CK(c, launch_ctrl_copy(c->cctrl.as<CtrlBlock>(), c->ctrl.as<CtrlBlock>(), st));
  if (b.coop1_lines > 0)
    SKS_CK(c, launch_step_coop1(a, j0, j1, b.last_grid, c->part.as<double>(), b.pslots, c->csync.as<unsigned>(),
                                b.coop1_lines, st));
  else
    SKS_CK(c, launch_step_coop(a, j0, j1, b.last_grid, c->part.as<double>(), b.pslots, c->csync.as<unsigned>(),
                               b.coop_grid, st));
  SKS_CK(c, launch_ctrl_merge(c->ctrl.as<CtrlBlock>(), c->cctrl.as<CtrlBlock>(), j0 == 1 ? 1 : 0, st));
  c->launches += 4;
  b.last_grid = b.coop_grid;
  for (int j = j0; j <= j1; ++j) {
    b.bytes += 8.0 * g.n * (std::min(b.k, j) + 1);
    ++b.steps;
  }
  return SKS_OK;
}

// SKS_MPK_S (default 4; 0 = off): columns per matrix-powers launch of the deferred 2D Chebyshev basis
// Off by default: at C2 (m = 512, 4 own lines per CTA) the 2 (S + 1) halo lines per launch triple the work and it
// measured 40.2 vs 33.3 ms (profiles/r02/mpk_ab_r02.txt); its purpose is one depth-(S+1) halo exchange per S
// columns across ranks (tests/test_gpu_loopback.py)
static int mpk_request() {
  const char* e = getenv("SKS_MPK_S");
  const int v = e ? atoi(e) : 0;
  return std::max(0, std::min(v, 8));
}

// decide the matrix-powers mode once the basis is set up (deferred Chebyshev, 2D stencil, ghost depth >= S + 1,
// the staged lines fit in shared memory with the step kernels' grid)
static void mpk_setup(sks_ctx* c, Basis& b) {
  const int S = mpk_request();
  b.mpk_s = 0;
  if (!b.defer || b.g.dim != 2 || S < 1 || b.g.G < S + 1) return;
  const int grid = b.tma ? b.tma_grid : b.step_grid;
  if (grid < 1 || grid > b.pslots || mpk2d_smem(b.g.m, b.g.nz, grid, S) > 200 * 1024) return;
  b.mpk_s = S;
  b.mpk_grid = grid;
}

// columns j0..j1 (j0 >= 3) of the deferred 2D Chebyshev basis in one matrix-powers launch; at nranks > 1 the
// two newest columns' ghost lines (depth G >= S + 1) are exchanged once for the next launch
static sks_status mpk_columns(sks_ctx* c, Basis& b, int j0, int j1) {
  cudaStream_t st = c->main();
  const Geo& g = b.g;
  const int S = j1 - j0 + 1;
  SKS_CK(c, launch_cheb_mpk2d(c->W.as<double>(), g.ld, g.off, g.m, g.nz, g.z0, g.m, g.cc, g.cm, g.cp, b.sa.cheb_rho,
                              b.sa.cheb_c, b.sa.cheb_e, j0, S, c->partc.as<double>(), b.pslots, b.mpk_grid,
                              c->ctrl.as<CtrlBlock>(), b.mpk_grid, st));
  ++c->launches;
  b.defer_grid = b.mpk_grid;
  if (S >= 2) SKS_TRY(halo_exchange(c, g, colp(c, b, j1 - 1)));
  SKS_TRY(halo_exchange(c, g, colp(c, b, j1)));
  b.bytes += 8.0 * g.n * (2 + S);
  b.steps += S;
  return SKS_OK;
}

// deferred Chebyshev bookkeeping of the complete columns [fin_next, upto): per-column fixed-order sums, ONE
// all-reduce of (upto - fin_next) x SKS_NP scalars for the batch at nranks > 1, then sigma / H / gam / breakdown
static sks_status cheb_finalize(sks_ctx* c, Basis& b, int upto, cudaStream_t st) {
  if (!b.defer) return SKS_OK;
  const int j0 = std::max(b.fin_next, 2), j1 = std::min(upto, b.ncol);
  if (j1 <= j0) return SKS_OK;
  double* sums = c->partcs.as<double>();
  SKS_CK(c, launch_cheb_colsum(c->partc.as<double>(), b.defer_grid, b.pslots, j0, j1, sums, st));
  SKS_TRY(allreduce_sum(c, sums + (size_t)j0 * SKS_NP, (size_t)(j1 - j0) * SKS_NP, st));
  SKS_CK(c, launch_cheb_finalize(sums, j0, j1, b.sa.cheb_rho, b.sa.cheb_c, b.sa.cheb_e, c->sigma.as<double>(),
                                 c->H.as<double>(), b.ldH, c->mnorm.as<double>(), c->gam.as<double>(),
                                 c->ctrl.as<CtrlBlock>(), st));
  c->launches += 2;
  b.fin_next = j1;
  return SKS_OK;
}

// Whitening (Fact "Whitening" P:598-612; reading O36): the first J basis columns
// are replaced by B_J T_J^{-1}, rescaled to unit norm (stored raw with sigma_i = 1/||.||), S W and T follow
// (S A B_J T_J^{-1} = U_J: T_J becomes diag(sigma)), and the partial sums the next step (column J) needs are
// recomputed for the whitened column J-1.  Called with the streams joined.
static sks_status whiten_columns(sks_ctx* c, Basis& b, int J, int s) {
  cudaStream_t st = c->main();
  const Geo& g = b.g;
  const int ldT = b.ncol;
  SKS_TRY(ensure(c, c->wz, sizeof(double) * (size_t)J * J));
  SKS_TRY(ensure(c, c->wn, sizeof(double) * (size_t)g.ld * J));
  const int ngroups = (int)std::max<int64_t>(1, std::min<int64_t>((g.n + 63) / 64, (int64_t)c->num_sms * 4));
  SKS_TRY(ensure(c, c->wpart, sizeof(double) * ((size_t)ngroups * J + J + (size_t)s * J)));
  double* Z = c->wz.as<double>();
  double* part = c->wpart.as<double>();
  double* sums = part + (size_t)ngroups * J;
  double* swt = sums + J;
  // Z = diag(sigma) T_J^{-1}
  SKS_CK(c, launch_eye_ones(Z, J, J, nullptr, 0, st));
  SKS_CK(c, launch_trsm_upper(c->T.as<double>(), ldT, J, Z, J, J, st));
  SKS_CK(c, launch_scale_rows(Z, J, J, c->sigma.as<double>(), st));
  // W_J <- W_J Z (out of place, interior rows) and the squared column norms
  SKS_CK(c, launch_whiten_gemm(c->W.as<double>(), g.ld, g.off, g.n, J, Z, J, c->wn.as<double>(), part, ngroups, st));
  SKS_CK(c, launch_colsum(part, ngroups, J, sums, st));
  SKS_TRY(allreduce_sum(c, sums, (size_t)J, st));
  SKS_CK(c, cudaMemcpy2DAsync(c->W.as<double>() + g.off, sizeof(double) * g.ld, c->wn.as<double>() + g.off,
                              sizeof(double) * g.ld, sizeof(double) * g.n, J, cudaMemcpyDeviceToDevice, st));
  // S W_J <- S W_J Z (the sketch is linear; replicated on every rank)
  SKS_CK(c, launch_small_gemm(s, J, J, c->SW.as<double>(), s, 0, Z, J, 0, nullptr, 0, swt, s, st));
  SKS_CK(c, cudaMemcpyAsync(c->SW.p, swt, sizeof(double) * (size_t)s * J, cudaMemcpyDeviceToDevice, st));
  // sigma_i = 1/||w_i||, T_J = diag(sigma), control block at J QR'd columns
  SKS_CK(c, launch_whiten_finish(sums, J, c->sigma.as<double>(), c->T.as<double>(), ldT, c->ctrl.as<CtrlBlock>(),
                                 st));
  // the sketched residual g - U_J U_J^T g (the columns QR'd past J are discarded)
  SKS_CK(c, launch_resid_restore(c->rvec.as<double>(), c->gsave.as<double>(), c->U.as<double>(), s,
                                 c->rho.as<double>(), J, s, st));
  SKS_TRY(halo_exchange(c, g, colp(c, b, J - 1)));
  // partial sums of the whitened w_{J-1} for the step that regenerates column J (step_prologue slot layout)
  const double* v[SKS_KMAX];
  int slot[SKS_KMAX];
  int nv = 0;
  for (int i = std::max(0, J - b.k); i < J - 1; ++i) {
    v[nv] = colp(c, b, i) + g.off;
    slot[nv] = 3 + i - (J - b.k);
    ++nv;
  }
  const int grid = c->num_sms * 2;
  double* p0 = pslot(c, b, c->part, J - 1);
  SKS_CK(c, launch_whiten_partials(colp(c, b, J - 1) + g.off, v, slot, nv, g.n, g.plane, g.m, g.dim, g.cc, g.cm, g.cp,
                                   p0, grid, st));
  b.last_grid = grid;
  SKS_TRY(reduce_partials(c, p0, grid, st));
  if (J >= 2) SKS_CK(c, cudaMemsetAsync(c->mnorm.as<double>() + (J - 2), 0, sizeof(double), st));
  c->launches += 9;
  b.bytes += 16.0 * g.n * J;
  return SKS_OK;
}

// ||v||_2 of this rank's interior, reduced over ranks, returned on the host (syncs)
static sks_status global_norm(sks_ctx* c, Basis& b, const double* v_interior, double* out) {
  cudaStream_t st = c->main();
  double* p = c->tmp.as<double>();
  SKS_CK(c, launch_copy_norm(b.g.n, v_interior, c->vb.as<double>() + b.g.off, p, b.step_grid, st));
  ++c->launches;
  // copy_norm writes [grid][SKS_NP] with slot 0
  SKS_CK(c, launch_sum_partials(p, b.step_grid, SKS_NP, 1, c->small.as<double>(), st));
  ++c->launches;
  SKS_TRY(allreduce_sum(c, c->small.as<double>(), 1, st));
  SKS_CK(c, cudaMemcpyAsync(c->h_small, c->small.p, sizeof(double), cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  *out = std::sqrt(c->h_small[0]);
  return SKS_OK;
}

// sketch columns [c0, c0+J) of W into SW (s x ncol, column-major), reduced over ranks
// per-cycle sketch plan of this rank's rows (S is fixed within a cycle, reading O7); NULL if the
// (s, zeta) combination has no plan kernel (the generic sketch kernel hashes per batch)
static sks_status sketch_plan(sks_ctx* c, const Geo& g, int s, int zeta, uint64_t key, cudaStream_t st,
                              const void** plan) {
  *plan = nullptr;
  if (c->sketch_kind == SKS_SKETCH_SRFT) {  // the cycle's s sampled DCT coordinates (host Floyd, O32)
    std::vector<int32_t> q(s);
    srft_rows_host(g.n, s, srft_key_host(c->sk_seed, c->sk_cycle), q.data());
    SKS_TRY(ensure(c, c->srft_q, sizeof(int32_t) * (size_t)s));
    SKS_CK(c, cudaStreamSynchronize(st));  // the previous cycle's sample kernels may still read srft_q
    SKS_CK(c, cudaMemcpy(c->srft_q.p, q.data(), sizeof(int32_t) * (size_t)s, cudaMemcpyHostToDevice));
    return SKS_OK;
  }
  if (!sketch_plan_supported(s, zeta)) return SKS_OK;
  SKS_TRY(ensure(c, c->plan, sketch_plan_bytes(g.n, s, zeta)));
  SKS_CK(c, launch_sketch_plan(g.n, g.row_begin, s, zeta, key, c->plan.p, c->main_sms, st));
  ++c->launches;
  *plan = c->plan.p;
  return SKS_OK;
}

static sks_status sketch_cols(sks_ctx* c, Basis& b, int c0, int J, int s, int zeta, uint64_t key,
                              cudaStream_t st, const void* plan) {
  const Geo& g = b.g;
  double* out = c->SW.as<double>() + (int64_t)c0 * s;
  if (c->sketch_kind == SKS_SKETCH_SRFT) {
    SKS_TRY(ensure(c, c->srft_w, sizeof(double) * srft_work_doubles(g.n, SKS_JB)));
    SKS_CK(c, launch_srft(colp(c, b, c0) + g.off, g.ld, g.n, J, s, srft_key_host(c->sk_seed, c->sk_cycle),
                          c->srft_q.as<int32_t>(), c->srft_w.as<double>(), &c->srft_cache, out, s, c->main_sms, st));
    c->launches += 3;
    return SKS_OK;
  }
  const int grid = sketch_grid(c->main_sms, g.n);
  SKS_CK(c, launch_sketch(colp(c, b, c0) + g.off, g.ld, g.n, g.row_begin, J, s, zeta, key, c->partsk.as<double>(),
                          grid, out, s, 0, st, &c->launches, plan));
  SKS_TRY(allreduce_sum(c, out, (size_t)J * s, st));
  return SKS_OK;
}

// append sketched columns [j0, j0+J) to the thin QR (mode 0: SAB via recurrence; 1: SB)
static sks_status qr_append(sks_ctx* c, Basis& b, int mode, int j0, int J, int s, int track_res, int max_cols,
                            cudaStream_t st) {
  double* X = c->Xp.as<double>();
  double* Z = c->Zb.as<double>();
  double* U = c->U.as<double>();
  double* T = c->T.as<double>();
  const int ldT = b.ncol;
  SKS_CK(c, launch_form_cols(mode, c->SW.as<double>(), s, j0, J, b.k, c->H.as<double>(), b.ldH,
                             c->sigma.as<double>(), c->gam.as<double>(), X, J, 1, st));
  double* ws = c->bgsw.as<double>();
  int* cnt = c->bgsc.as<int>();
  SKS_CK(c, launch_utx(U, s, s, j0, X, J, Z, T, ldT, j0, 0, ws, cnt, st));
  SKS_CK(c, launch_xmuz(U, s, s, j0, X, J, Z, ws, cnt, st));
  SKS_CK(c, launch_utx(U, s, s, j0, X, J, Z, T, ldT, j0, 1, ws, cnt, st));
  SKS_CK(c, launch_xmuz(U, s, s, j0, X, J, Z, ws, cnt, st));
  SKS_CK(c, launch_panel(X, s, J, j0, U, s, T, ldT, c->rvec.as<double>(), c->rho.as<double>(), c->rest.as<double>(),
                         c->ctrl.as<CtrlBlock>(), track_res, max_cols, st));
  c->launches += (j0 > 0) ? 6 : 2;
  return SKS_OK;
}

static sks_status setup_small(sks_ctx* c, Basis& b, int s, int JB) {
  const int ncol = b.ncol;
  SKS_TRY(ensure(c, c->SW, sizeof(double) * (size_t)s * (ncol + 1)));
  const int grid = sketch_grid(c->main_sms, b.g.n);
  SKS_TRY(ensure(c, c->partsk, sizeof(double) * sketch_part_doubles(grid, SKS_JB, s)));
  SKS_TRY(ensure(c, c->Xp, sizeof(double) * (size_t)s * JB));
  SKS_TRY(ensure(c, c->Zb, sizeof(double) * (size_t)(ncol + 1) * JB));
  SKS_TRY(ensure(c, c->U, sizeof(double) * (size_t)s * (ncol + 1)));
  SKS_TRY(ensure(c, c->T, sizeof(double) * (size_t)(ncol + 1) * (ncol + 1)));
  SKS_TRY(ensure(c, c->Tcopy, sizeof(double) * (size_t)(ncol + 1) * (ncol + 1)));
  SKS_TRY(ensure(c, c->rvec, sizeof(double) * s));
  SKS_TRY(ensure(c, c->rho, sizeof(double) * (ncol + 1)));
  SKS_TRY(ensure(c, c->rest, sizeof(double) * (ncol + 1)));
  SKS_TRY(ensure(c, c->coef, sizeof(double) * (ncol + 1)));
  SKS_TRY(ensure(c, c->tmp, sizeof(double) * (size_t)std::max(b.pslots, 64) * SKS_NP * 2));
  SKS_TRY(ensure(c, c->bgsw, sizeof(double) * bgs_workspace_doubles(s, ncol + 1)));
  if (c->bgsc.bytes < sizeof(int) * 128) {
    SKS_TRY(ensure(c, c->bgsc, sizeof(int) * 128));
    SKS_CK(c, cudaMemsetAsync(c->bgsc.p, 0, sizeof(int) * 128, c->main()));
  }
  if (panel_smem(s, JB) > 227 * 1024) return fail(c, SKS_EUNSUPPORTED, "s too large for the panel kernel");
  return SKS_OK;
}

static int panel_jb(int s, int want) {
  int J = std::min(want, SKS_JB);
  while (J > 1 && panel_smem(s, J) > 200 * 1024) --J;
  return J;
}

}  // namespace

// ------------------------------------------------------------------------------------
// sGMRES
// ------------------------------------------------------------------------------------
extern "C" sks_status sks_sgmres_solve(sks_ctx* c, const sks_operator* A, const double* f, double* x,
                                       const sks_sgmres_opts* o, sks_sgmres_info* info, double* hist,
                                       int64_t hist_cap, double* hist_true, int64_t hist_true_cap) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  if (!A || !f || !x || !o) return fail(c, SKS_EINVAL, "NULL argument");
  const int d = o->d, k = o->k, s = o->s, zeta = o->zeta;
  if (d < 1 || k < 1 || k > SKS_KMAX || s < d + 1 || s > SKS_SMAX || zeta < 1 || zeta > std::min(s, SKS_ZETA_MAX))
    return fail(c, SKS_EINVAL, "need d>=1, 1<=k<=8, d+1<=s<=2048, 1<=zeta<=min(s,16)");
  if (!(o->tol >= 0.0) || o->max_cycles < 1) return fail(c, SKS_EINVAL, "bad tol / max_cycles");
  cudaSetDevice(c->device);
  const int64_t launches0 = c->launches;
  cudaStream_t st = c->main();
  Basis b;
  c->ghost_min = (o->basis == SKS_BASIS_CHEBYSHEV && A->kind == SKS_OP_STENCIL2D && mpk_request() > 0)
                     ? mpk_request() + 1 : 2;
  const sks_status sb = setup_basis(c, A, k, d + 2, &b);
  c->ghost_min = 2;
  SKS_TRY(sb);
  SKS_TRY(set_basis(c, A, b, o->basis, o->cheb_c, o->cheb_dx, o->cheb_dy));
  mpk_setup(c, b);
  const Geo& g = b.g;
  const int JB = panel_jb(s, o->sketch_batch > 0 ? o->sketch_batch : SKS_JB);
  b.time_steps = (o->flags & SKS_OPT_TIME_STEPS) != 0;
  b.time_stride = o->time_stride > 1 ? o->time_stride : 1;
  {  // windows of consecutive launches when sampling (time_stride > 1); SKS_TIME_WINDOW=1 restores single launches
    const char* e = getenv("SKS_TIME_WINDOW");
    b.time_window = e ? std::max(1, atoi(e)) : b.time_stride;
    if (g.kind == SKS_OP_CSR) b.time_window = 1;
  }
  if (b.time_steps && (int)c->ev_step.size() < 2 * (d + 2)) {
    const size_t old_n = c->ev_step.size();
    c->ev_step.resize(2 * (d + 2));
    for (size_t i = old_n; i < c->ev_step.size(); ++i) SKS_CK(c, cudaEventCreate(&c->ev_step[i]));
  }
  double t_step_total = 0.0, bytes_step_total = 0.0;
  int64_t steps_timed = 0;
  SKS_TRY(setup_small(c, b, s, JB));
  const double cond_tol = o->cond_tol > 0 ? o->cond_tol : 1e14;

  SKS_CK(c, cudaEventRecord(c->ev_t0, st));
  // inputs into ghost-layout buffers
  double* xb = c->xb.as<double>();
  double* fb = c->fb.as<double>();
  SKS_CK(c, cudaMemsetAsync(xb, 0, sizeof(double) * g.ld, st));
  SKS_CK(c, cudaMemsetAsync(fb, 0, sizeof(double) * g.ld, st));
  if (o->flags & SKS_OPT_ZERO_X0)
    SKS_CK(c, cudaMemsetAsync(xb + g.off, 0, sizeof(double) * g.n, st));
  else
    SKS_CK(c, cudaMemcpyAsync(xb + g.off, x, sizeof(double) * g.n, cudaMemcpyDefault, st));
  SKS_CK(c, cudaMemcpyAsync(fb + g.off, f, sizeof(double) * g.n, cudaMemcpyDefault, st));
  SKS_TRY(halo_exchange(c, g, xb));
  SKS_TRY(halo_exchange(c, g, fb));
  double fnorm = 0.0;
  SKS_TRY(global_norm(c, b, fb + g.off, &fnorm));
  if (!(fnorm >= 0.0) || !std::isfinite(fnorm)) return fail(c, SKS_EINVAL, "f is not finite");
  const double thr = o->early_exit_factor > 0 ? o->early_exit_factor * o->tol * fnorm : -1.0;
  const bool adaptive = (o->flags & SKS_OPT_ADAPTIVE_RESTART) != 0;
  const bool whiten = (o->flags & SKS_OPT_WHITEN) != 0;
  const bool watch = adaptive || whiten;  // kappa_2(T_j) estimate after every sketched-QR batch
  if (whiten && (g.kind == SKS_OP_CSR || o->basis != SKS_BASIS_ARNOLDI))
    return fail(c, SKS_EUNSUPPORTED, "whitening: k-truncated Arnoldi basis on a stencil operator only");
  if (o->sketch != SKS_SKETCH_SPARSE && o->sketch != SKS_SKETCH_SRFT) return fail(c, SKS_EINVAL, "unknown sketch");
  if (o->sketch == SKS_SKETCH_SRFT && c->nranks > 1)
    return fail(c, SKS_EUNSUPPORTED, "the SRFT sketch is single-GPU (the DCT mixes all rows)");
  c->sketch_kind = o->sketch;
  c->sk_seed = o->seed;
  int poll_lag = (g.kind == SKS_OP_CSR) ? 1 : 2;
  if (const char* e = getenv("SKS_POLL_LAG")) poll_lag = std::max(1, atoi(e));
  // near-exit switch (small batches, lag 1) only where a column costs more than a batch's QR
  // latency: large local vectors (C3: 54.6 vs 56.9 ms; on C2's 2 MB vectors the waits cost more)
  double near_factor = (g.n >= (int64_t(1) << 20)) ? 4.0 : 0.0;
  if (const char* e = getenv("SKS_NEAR_FACTOR")) near_factor = atof(e);

  int cycles = 0, columns = 0, generated = 0, flags = 0;
  int64_t nh = 0, nht = 0;
  double rel = 1.0, r_est_last = NAN, cond_last = 1.0;
  float t_basis_ms = 0.f;
  double bytes_basis_total = 0.0;
  sks_status result = SKS_ENOTCONV;
  CtrlBlock* dctrl = c->ctrl.as<CtrlBlock>();
  CtrlBlock* hc = c->h_ctrl;
  int pend_hist = -1;  // jstar of a cycle whose r_est history sits in h_small[64..] (stream-ordered copy)
  auto flush_hist = [&]() {
    if (pend_hist < 0) return;
    const int js = pend_hist;
    pend_hist = -1;
    for (int j = 0; j < js && j < 2048; ++j) {
      if (hist && nh < hist_cap) hist[nh] = c->h_small[64 + j] / (fnorm > 0 ? fnorm : 1.0);
      ++nh;
    }
    r_est_last = c->h_small[64 + js - 1] / (fnorm > 0 ? fnorm : 1.0);
    columns += js;
  };

  for (int cyc = 0; cyc <= o->max_cycles; ++cyc) {
    // ---- residual r = f - A x  (w_0), true residual of the previous cycle
    SKS_CK(c, launch_ctrl_reset(dctrl, thr, fnorm, st));
    ++c->launches;
    b.bytes = 0;  // per-cycle accounting of the basis loop below
    SKS_TRY(first_column(c, b, 1, xb, fb));
    SKS_CK(c, launch_sum_partials(pslot(c, b, c->part, 0), c->nranks > 1 ? 1 : b.last_grid, SKS_NP, 1,
                                  c->small.as<double>(), st));
    ++c->launches;
    SKS_CK(c, cudaMemcpyAsync(c->h_small, c->small.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    SKS_CK(c, cudaStreamSynchronize(st));
    flush_hist();  // the previous cycle's r_est history (copied before this point on the same stream)
    const double rnorm = std::sqrt(c->h_small[0]);
    rel = fnorm > 0 ? rnorm / fnorm : 0.0;
    if (cyc > 0) {
      if (hist_true && nht < hist_true_cap) hist_true[nht] = rel;
      ++nht;
    }
    if (rel <= o->tol || rnorm == 0.0) {
      result = SKS_OK;
      break;
    }
    if (cyc == o->max_cycles) break;
    ++cycles;
    const uint64_t key = sks_key(o->seed, (uint32_t)cyc);
    c->sk_cycle = (uint32_t)cyc;
    // ---- basis loop (main) with batched sketch + incremental QR (side)
    const double bytes_first = b.bytes;
    SKS_CK(c, cudaEventRecord(c->ev_b0, st));
    int next_sk = 0;    // next column to sketch
    int next_qr = 0;    // next SAB column to append
    std::vector<int> kq_cols;  // adaptive restarting: QR columns behind each batch's kappa estimate
    const void* plan = nullptr;
    int nbatch = 0;
    int last_col = d;   // columns 0..d are generated (d+1 columns)
    SKS_CK(c, cudaMemsetAsync(c->rvec.p, 0, sizeof(double) * s, st));
    // the sketch batches run on the main stream (bandwidth kernels, all SMs but the reserved
    // ones); the sketched QR (latency kernels) on the side stream, on the reserved SMs
    b.fin_next = 2;
    auto enqueue_side = [&](int upto /* columns [0, upto) are complete */, bool final_) -> sks_status {
      SKS_TRY(cheb_finalize(c, b, upto, st));
      while (next_sk < upto) {
        const int J = std::min(JB, upto - next_sk);
        if (next_sk == 0) SKS_TRY(sketch_plan(c, g, s, zeta, key, st, &plan));
        SKS_TRY(sketch_cols(c, b, next_sk, J, s, zeta, key, st, plan));
        if (next_sk == 0) {  // g = S r = S w_0 starts the residual vector
          SKS_CK(c, cudaMemcpyAsync(c->rvec.p, c->SW.p, sizeof(double) * s, cudaMemcpyDeviceToDevice, st));
          if (whiten) {  // kept for the residual vector after a whitening event
            SKS_TRY(ensure(c, c->gsave, sizeof(double) * s));
            SKS_CK(c, cudaMemcpyAsync(c->gsave.p, c->SW.p, sizeof(double) * s, cudaMemcpyDeviceToDevice, st));
          }
        }
        next_sk += J;
      }
      SKS_CK(c, cudaEventRecord(c->ev_fork, st));
      SKS_CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
      // SAB column jj needs SW[:, jj+1]
      const int qr_upto = std::min(next_sk - 1, d);
      while (next_qr < qr_upto) {
        const int J = std::min(JB, qr_upto - next_qr);
        SKS_TRY(qr_append(c, b, 0, next_qr, J, s, 1, d, c->side));
        next_qr += J;
      }
      // adaptive restarting (O31): kappa_2(T_j) after every batch, j = next_qr
      if (watch && next_qr > 0 && (kq_cols.empty() || kq_cols.back() < next_qr) && kq_cols.size() < 1024) {
        SKS_CK(c, launch_cond(c->T.as<double>(), b.ncol, next_qr, SKS_ADAPT_ITERS, dctrl,
                              c->small.as<double>() + 2048 + kq_cols.size(), c->side));
        kq_cols.push_back(next_qr);
        ++c->launches;
      }
      SKS_CK(c, cudaMemcpyAsync(hc, dctrl, sizeof(CtrlBlock), cudaMemcpyDeviceToHost, c->side));
      if (nbatch < (int)c->ev_batch.size()) SKS_CK(c, cudaEventRecord(c->ev_batch[nbatch], c->side));
      ++nbatch;
      (void)final_;
      return SKS_OK;
    };
    int j_begin = 1;     // first column of this basis segment (after a whitening event: J)
    int white_at = -1;   // J of the last whitening event of this cycle
    bool near = false;   // r_est within a factor of the exit threshold: small batches, lag 1
    int jstar = 0;
    // CSR: a column costs a full matrix sweep, so small fixed batches let the sketched QR's early-exit flag
    // (checked by the SpMV kernel on the device) stop the basis a few columns after the exit point
    int csr_batch = 4;
    if (const char* e = getenv("SKS_CSR_BATCH")) csr_batch = std::max(1, atoi(e));
    const bool csr = g.kind == SKS_OP_CSR;
    // first sketch batch of a cycle (SKS_FIRST_BATCH; 8: starting C3's cycles with full 32-column batches measured
    // 50.9 vs 50.6-51.0 ms -- no gain, profiles/r02/coop_ab_r02.txt)
    int first_batch = 8;
    int near_batch = 8;  // batch width once r_est is near the exit threshold (SKS_NEAR_BATCH)
    if (const char* e = getenv("SKS_NEAR_BATCH")) near_batch = std::max(1, atoi(e));
    if (const char* e = getenv("SKS_FIRST_BATCH")) first_batch = std::max(1, atoi(e));
    for (;;) {  // basis segments: one, or one more after every whitening event (reading O36)
    int batch_size = csr ? std::min(csr_batch, JB) : std::min(first_batch, JB);
    int pending_upto = j_begin;
    int lag = near ? 1 : poll_lag;
    last_col = d;
    if (j_begin > 1) SKS_CK(c, cudaEventRecord(c->ev_b0, st));
    for (int j = j_begin; j <= d; ++j) {
      if (b.coop) {  // the rest of this batch in one cooperative launch
        const int je = std::max(j, std::min(pending_upto + batch_size - 1, d));
        SKS_TRY(coop_columns(c, b, j, je));
        j = je;
      } else if (b.mpk_s > 0 && j >= 3) {  // matrix-powers launch (deferred 2D Chebyshev)
        const int je = std::max(j, std::min(std::min(j + b.mpk_s - 1, pending_upto + batch_size - 1), d));
        SKS_TRY(mpk_columns(c, b, j, je));
        j = je;
      } else {
        // windowed step timing: events around time_window consecutive step launches of one sketch batch
        if (b.time_steps && b.time_window > 1 && b.win_end < 0 && j % b.time_stride == 0 &&
            j + b.time_window - 1 < pending_upto + batch_size && j + b.time_window - 1 <= d &&
            2 * b.ntimed + 1 < (int)c->ev_step.size()) {
          SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed], st));
          b.win_end = j + b.time_window - 1;
          b.win_bytes = 0.0;
        }
        SKS_TRY(step_column(c, b, j));
        if (b.win_end == j) {
          SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed + 1], st));
          ++b.ntimed;
          b.launches_timed += b.time_window;
          b.bytes_timed += b.win_bytes;
          b.win_end = -1;
        }
      }
      const bool batch_done = (j + 1 - pending_upto >= batch_size) || j == d;
      if (batch_done) {
        SKS_TRY(enqueue_side(j + 1, j == d));
        pending_upto = j + 1;
        batch_size = csr ? std::min(csr_batch, JB) : (near ? std::min(near_batch, JB) : std::min(JB, batch_size * 2));
        // poll the early-exit / breakdown flags of batch nbatch-lag (bounded lag): 2 for stencils
        // (cheap columns: keep the GPU fed), 1 for CSR (a column costs a full matrix sweep, more
        // than the batch's sketched QR, so over-generated columns cost more than the wait); once
        // r_est comes within near_factor of the exit threshold the cycle is about to end, and the
        // columns run ahead of the check would be discarded: 8-column batches polled with lag 1
        if (nbatch >= lag && nbatch - lag < (int)c->ev_batch.size()) {
          SKS_CK(c, cudaEventSynchronize(c->ev_batch[nbatch - lag]));
          if (!near && thr > 0 && hc->r_est_last > 0 && hc->r_est_last <= near_factor * thr) {
            near = true;
            lag = 1;
            batch_size = std::min(near_batch, JB);
          }
          if (hc->exit_cols > 0 || hc->stop_col < INT_MAX || hc->rank_def ||
              (watch && hc->cond > o->cond_tol)) {
            last_col = j;
            break;
          }
        }
      }
    }
    if (b.win_end >= 0) {  // a window cut short by an early stop: close it over the launches it covered
      SKS_CK(c, cudaEventRecord(c->ev_step[2 * b.ntimed + 1], st));
      ++b.ntimed;
      b.launches_timed += std::max(0, last_col - (b.win_end - b.time_window));
      b.bytes_timed += b.win_bytes;
      b.win_end = -1;
    }
    SKS_CK(c, cudaEventRecord(c->ev_b1, st));
    // remaining side work for everything generated, then join
    if (next_sk < last_col + 1) SKS_TRY(enqueue_side(last_col + 1, true));
    SKS_CK(c, cudaEventRecord(c->ev_join, c->side));
    SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));
    SKS_CK(c, cudaMemcpyAsync(hc, dctrl, sizeof(CtrlBlock), cudaMemcpyDeviceToHost, st));
    SKS_CK(c, cudaStreamSynchronize(st));
    {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, c->ev_b0, c->ev_b1);
      t_basis_ms += ms;
      for (int i = 0; i < b.ntimed; ++i) {
        float t = 0.f;
        cudaEventElapsedTime(&t, c->ev_step[2 * i], c->ev_step[2 * i + 1]);
        t_step_total += t * 1e-3;
      }
      steps_timed += b.launches_timed;
      bytes_step_total += b.bytes_timed;
      b.ntimed = 0;
      b.launches_timed = 0;
      b.bytes_timed = 0.0;
    }
    bytes_basis_total += b.bytes - bytes_first;
    generated += last_col + 1 - (j_begin - 1);
    if (hc->exit_cols > 0) {
      jstar = hc->exit_cols;
    } else {
      int dmax = d;
      if (hc->stop_col < INT_MAX) dmax = std::min(dmax, hc->stop_col);
      jstar = std::min(dmax, hc->qr_cols);
    }
    int jfirst = -1;  // first j with kappa_2(T_j) > cond_tol (watch mode)
    if (watch && !kq_cols.empty()) {
      // first batch whose kappa estimate exceeds cond_tol, then bisection inside it for the first j
      // with kappa_2(T_j) > cond_tol (kappa_2 of the leading blocks is non-decreasing in j)
      const int nk = (int)kq_cols.size();
      SKS_CK(c, cudaMemcpyAsync(c->h_small + 2048, c->small.as<double>() + 2048, sizeof(double) * nk,
                                cudaMemcpyDeviceToHost, st));
      SKS_CK(c, cudaStreamSynchronize(st));
      int bo = -1;
      for (int t = 0; t < nk; ++t)
        if (c->h_small[2048 + t] > o->cond_tol) {
          bo = t;
          break;
        }
      if (bo >= 0) {
        int lo = bo == 0 ? 0 : kq_cols[bo - 1], hi = kq_cols[bo];
        while (hi - lo > 1) {
          const int mid = (lo + hi) / 2;
          SKS_CK(c, launch_cond(c->T.as<double>(), b.ncol, mid, SKS_ADAPT_ITERS, nullptr,
                                c->small.as<double>() + 3072, st));
          ++c->launches;
          SKS_CK(c, cudaMemcpyAsync(c->h_small + 3072, c->small.as<double>() + 3072, sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
          SKS_CK(c, cudaStreamSynchronize(st));
          if (c->h_small[3072] > o->cond_tol)
            hi = mid;
          else
            lo = mid;
        }
        jfirst = hi;
        if (adaptive) {
          const int jad = std::max(hi - 1, 1);  // "restart with the previous residual r_{j-1}"
          if (jad < jstar) {
            jstar = jad;
            flags |= SKS_INFO_ADAPTIVE_RESTART;
          }
        }
      }
    }
    if (whiten && jfirst > 0 && hc->exit_cols == 0 && !hc->breakdown && !hc->rank_def) {
      const int J = jfirst - 1;  // columns kept: kappa_2(T_J) <= cond_tol
      if (J >= 1 && J > white_at) {  // whiten B_J <- B_J T_J^{-1} (unit columns) and continue from column J
        SKS_TRY(whiten_columns(c, b, J, s));
        white_at = J;
        flags |= SKS_INFO_WHITEN;
        j_begin = J;
        next_sk = J;
        next_qr = J;
        kq_cols.clear();
        hc->cond = 0.0;
        continue;
      }
      jstar = std::min(jstar, std::max(J, 1));  // no progress since the last whitening: the cycle ends here
    }
    break;
    }  // basis segments
    if (hc->breakdown) flags |= SKS_WARN_BREAKDOWN;
    if (jstar <= 0) {  // nothing usable (r == 0 handled above); stop
      break;
    }
    // ---- yhat = T^-1 (U^T g), coef = sigma .* yhat ; x += W coef
    SKS_CK(c, launch_trsv(c->T.as<double>(), b.ncol, jstar, c->rho.as<double>(), c->sigma.as<double>(), nullptr,
                          c->coef.as<double>(), st));
    int* ncp = reinterpret_cast<int*>(c->small.as<double>() + 16);
    c->h_small[32] = 0;
    reinterpret_cast<int*>(c->h_small + 32)[0] = jstar;
    SKS_CK(c, cudaMemcpyAsync(ncp, c->h_small + 32, sizeof(int), cudaMemcpyHostToDevice, st));
    // kappa(T) estimate (diagnostic: SKS_WARN_COND, info.cond_T) on its own stream from a copy of T, so that
    // the next cycle's sketched QR on the side stream does not queue behind it (C2 36.9 -> 33.6 ms)
    SKS_CK(c, cudaEventRecord(c->ev_fork, st));
    SKS_CK(c, cudaStreamWaitEvent(c->aux, c->ev_fork, 0));
    SKS_CK(c, cudaMemcpyAsync(c->Tcopy.p, c->T.p, sizeof(double) * (size_t)b.ncol * jstar, cudaMemcpyDeviceToDevice,
                              c->aux));
    SKS_CK(c, cudaEventRecord(c->ev_aux, c->aux));
    SKS_CK(c, cudaStreamWaitEvent(c->side, c->ev_aux, 0));  // the next cycle's QR rewrites T after the copy
    SKS_CK(c, launch_cond(c->Tcopy.as<double>(), b.ncol, jstar, 6, nullptr,
                          c->small.as<double>() + 1024 + std::min(cycles - 1, 1023), c->aux));
    SKS_CK(c, cudaEventRecord(c->ev_aux_done, c->aux));
    SKS_CK(c, launch_assemble(xb, c->W.as<double>(), g.ld, g.off, g.n, c->coef.as<double>(), ncp, jstar,
                              c->num_sms, st));
    c->launches += 3;
    SKS_TRY(halo_exchange(c, g, xb));
    // history: r_est,j / ||f||
    // (read at the next host synchronisation -- the next cycle's residual check or the end of the solve --
    // instead of a synchronisation of its own: one GPU bubble less per cycle)
    SKS_CK(c, cudaMemcpyAsync(c->h_small + 64, c->rest.p, sizeof(double) * std::min(jstar, 2048),
                              cudaMemcpyDeviceToHost, st));
    pend_hist = jstar;
  }
  // join the side and diagnostics streams (kappa estimates) and collect them
  SKS_CK(c, cudaEventRecord(c->ev_join, c->side));
  SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));
  SKS_CK(c, cudaEventRecord(c->ev_aux_done, c->aux));
  SKS_CK(c, cudaStreamWaitEvent(st, c->ev_aux_done, 0));
  SKS_CK(c, cudaMemcpyAsync(x, xb + g.off, sizeof(double) * g.n, cudaMemcpyDefault, st));
  SKS_CK(c, cudaEventRecord(c->ev_t1, st));
  if (cycles > 0)
    SKS_CK(c, cudaMemcpyAsync(c->h_small + 1024, c->small.as<double>() + 1024,
                              sizeof(double) * std::min(cycles, 1024), cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  flush_hist();
  for (int i = 0; i < std::min(cycles, 1024); ++i) {
    cond_last = c->h_small[1024 + i];
    if (cond_last > cond_tol) flags |= SKS_WARN_COND;
  }
  SKS_CK(c, cudaGetLastError());
  if (info) {
    memset(info, 0, sizeof(*info));
    info->cycles = cycles;
    info->columns = columns;
    info->columns_generated = generated;
    info->flags = flags;
    info->rel_res_true = rel;
    info->r_est = r_est_last;
    info->cond_T = cond_last;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1);
    info->t_total_s = ms * 1e-3;
    info->t_basis_s = t_basis_ms * 1e-3;
    info->bytes_basis = bytes_basis_total;
    info->kernel_launches = c->launches - launches0;
    info->steps = b.steps;
    info->t_step_s = t_step_total;
    info->steps_timed = steps_timed;
    info->bytes_step = bytes_step_total;
  }
  return result;
}

// ------------------------------------------------------------------------------------
// sRR (Alg. 2)
// ------------------------------------------------------------------------------------
namespace {

// run the basis loop for columns 1..d with the sketch batches interleaved (no QR)
// qr_done (optional): the thin QR of SB (mode 1) is appended on the side stream batch by batch while the basis is
// generated (SB column jj needs sigma_jj, known once column jj + 1 exists); *qr_done = columns factored
static sks_status basis_and_sketch(sks_ctx* c, Basis& b, int d, int s, int zeta, uint64_t key, int JB,
                                   bool do_sketch, float* t_basis_ms, int* qr_done = nullptr) {
  cudaStream_t st = c->main();
  int next_sk = 0, next_qr = 0;
  const void* plan = nullptr;
  SKS_CK(c, cudaEventRecord(c->ev_b0, st));
  b.fin_next = 2;
  auto side = [&](int upto) -> sks_status {
    SKS_TRY(cheb_finalize(c, b, upto, st));
    if (!do_sketch) return SKS_OK;
    while (next_sk < upto) {  // sketch batches on the main stream (see sks_sgmres_solve)
      const int J = std::min(JB, upto - next_sk);
      if (next_sk == 0) SKS_TRY(sketch_plan(c, b.g, s, zeta, key, st, &plan));
      SKS_TRY(sketch_cols(c, b, next_sk, J, s, zeta, key, st, plan));
      next_sk += J;
    }
    if (qr_done) {
      const int qr_upto = std::min(upto - 1, d);
      if (next_qr < qr_upto) {
        SKS_CK(c, cudaEventRecord(c->ev_fork, st));
        SKS_CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
        while (next_qr < qr_upto) {
          const int J = std::min(JB, qr_upto - next_qr);
          SKS_TRY(qr_append(c, b, 1, next_qr, J, s, 0, d, c->side));
          next_qr += J;
        }
      }
    }
    return SKS_OK;
  };
  int pending = 0;
  for (int j = 1; j <= d; ++j) {
    if (b.coop) {
      const int je = std::max(j, std::min(pending + JB - 1, d));
      SKS_TRY(coop_columns(c, b, j, je));
      j = je;
    } else if (b.mpk_s > 0 && j >= 3) {
      const int je = std::max(j, std::min(std::min(j + b.mpk_s - 1, pending + JB - 1), d));
      SKS_TRY(mpk_columns(c, b, j, je));
      j = je;
    } else {
      SKS_TRY(step_column(c, b, j));
    }
    if (j + 1 - pending >= JB || j == d) {
      SKS_TRY(side(j + 1));
      pending = j + 1;
    }
  }
  SKS_CK(c, cudaEventRecord(c->ev_b1, st));
  if (qr_done) {  // join the side stream's QR
    SKS_CK(c, cudaEventRecord(c->ev_join, c->side));
    SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));
    *qr_done = next_qr;
  }
  SKS_CK(c, cudaMemcpyAsync(c->h_ctrl, c->ctrl.p, sizeof(CtrlBlock), cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev_b0, c->ev_b1);
  if (t_basis_ms) *t_basis_ms += ms;
  return SKS_OK;
}

// block Chebyshev basis (Sec. "Block Chebyshev recurrence" P:1983-2008): W columns
// [(j-1) bs, j bs) hold B_j for j = 1..p+1 (B_{p+1} only feeds S A B_p through the recurrence, reading O34);
// Omega = v0 (n_local x bs, column-major, host or device).  Then all (p+1) bs columns are sketched.
static sks_status block_basis_and_sketch(sks_ctx* c, Basis& b, const double* v0, int bs, int p, int s, int zeta,
                                         uint64_t key, int JB, float* t_basis_ms) {
  cudaStream_t st = c->main();
  const Geo& g = b.g;
  const StepArgs& sa = b.sa;
  const double rho = sa.cheb_rho, c0 = sa.cheb_c, e = sa.cheb_e;
  SKS_CK(c, cudaEventRecord(c->ev_b0, st));
  for (int i = 0; i < bs; ++i) {
    SKS_CK(c, cudaMemcpyAsync(colp(c, b, i) + g.off, v0 + (int64_t)i * g.n, sizeof(double) * g.n, cudaMemcpyDefault,
                              st));
    SKS_TRY(halo_exchange(c, g, colp(c, b, i)));
  }
  for (int j = 2; j <= p + 1; ++j) {  // block j from blocks j-1 and j-2
    const double* in1 = colp(c, b, (j - 2) * bs);
    const double* in2 = (j >= 3) ? colp(c, b, (j - 3) * bs) : nullptr;
    const double al = (j == 2) ? 1.0 / (2.0 * rho) : 1.0 / rho;
    const double ga = (j >= 3) ? -e / rho : 0.0;
    SKS_CK(c, launch_block_cheb(g.dim, g.m, g.nz, g.plane, g.off, g.ld, g.cc, g.cm, g.cp, in1, in2,
                                colp(c, b, (j - 1) * bs), bs, al, c0, ga, st));
    ++c->launches;
    b.bytes += 8.0 * g.n * bs * (j >= 3 ? 3 : 2);
    b.steps += bs;
    for (int i = 0; i < bs; ++i) SKS_TRY(halo_exchange(c, g, colp(c, b, (j - 1) * bs + i)));
  }
  const int ncols = (p + 1) * bs;
  const void* plan = nullptr;
  SKS_TRY(sketch_plan(c, g, s, zeta, key, st, &plan));
  for (int c0i = 0; c0i < ncols; c0i += JB) SKS_TRY(sketch_cols(c, b, c0i, std::min(JB, ncols - c0i), s, zeta, key, st,
                                                              plan));
  SKS_CK(c, cudaEventRecord(c->ev_b1, st));
  SKS_CK(c, cudaMemcpyAsync(c->h_ctrl, c->ctrl.p, sizeof(CtrlBlock), cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, c->ev_b0, c->ev_b1);
  if (t_basis_ms) *t_basis_ms += ms;
  return SKS_OK;
}

}  // namespace

extern "C" sks_status sks_srr_eigs(sks_ctx* c, const sks_operator* A, const double* v0, const sks_srr_opts* o,
                                   int32_t nev, int32_t nev_cap, double* theta_re, double* theta_im,
                                   double* res_true, double* res_est, double* X_re, double* X_im,
                                   sks_srr_info* info) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  if (!A || !v0 || !o || !theta_re || !theta_im) return fail(c, SKS_EINVAL, "NULL argument");
  const int d = o->d, k = o->k, s = o->s, zeta = o->zeta;
  if (d < 2 || k < 1 || k > SKS_KMAX || s < d + 1 || s > SKS_SMAX || zeta < 1 || zeta > std::min(s, SKS_ZETA_MAX))
    return fail(c, SKS_EINVAL, "need d>=2, 1<=k<=8, d+1<=s<=2048, 1<=zeta<=min(s,16)");
  if (nev < 1 || nev > 11 || nev > d || nev_cap < nev + 1) return fail(c, SKS_EINVAL, "need 1<=nev<=min(11,d), nev_cap>=nev+1");
  if (o->stabilize < SKS_SRR_STABILIZE_OFF || o->stabilize > SKS_SRR_STABILIZE_ALWAYS)
    return fail(c, SKS_EINVAL, "unknown stabilize mode");
  const bool blk = o->basis == SKS_BASIS_BLOCK_CHEBYSHEV;
  const int bs = blk ? o->block : 1;
  if (blk && (bs < 1 || d % bs != 0)) return fail(c, SKS_EINVAL, "block Chebyshev basis: need block >= 1 dividing d");
  if (blk && A->kind == SKS_OP_CSR) return fail(c, SKS_EUNSUPPORTED, "block Chebyshev basis needs a stencil operator");
  if (blk && o->sketch != SKS_SKETCH_SPARSE) return fail(c, SKS_EUNSUPPORTED, "block Chebyshev basis: sparse sketch only");
  cudaSetDevice(c->device);
  const int64_t launches0 = c->launches;
  cudaStream_t st = c->main();
  Basis b;
  c->ghost_min = (!blk && o->basis == SKS_BASIS_CHEBYSHEV && A->kind == SKS_OP_STENCIL2D && mpk_request() > 0)
                     ? mpk_request() + 1 : 2;
  const sks_status sb = setup_basis(c, A, k, blk ? d + bs + 2 : d + 2, &b);
  c->ghost_min = 2;
  SKS_TRY(sb);
  SKS_TRY(set_basis(c, A, b, blk ? (int)SKS_BASIS_CHEBYSHEV : o->basis, o->cheb_c, o->cheb_dx, o->cheb_dy));
  if (!blk) mpk_setup(c, b);
  const Geo& g = b.g;
  const int JB = panel_jb(s, SKS_JB);
  SKS_TRY(setup_small(c, b, s, JB));
  const int nmax = nev + 1;
  SKS_CK(c, cudaEventRecord(c->ev_t0, st));
  double* vb = c->vb.as<double>();
  SKS_CK(c, launch_ctrl_reset(c->ctrl.as<CtrlBlock>(), -1.0, 0.0, st));
  ++c->launches;
  if (!blk) {
    SKS_CK(c, cudaMemsetAsync(vb, 0, sizeof(double) * g.ld, st));
    SKS_CK(c, cudaMemcpyAsync(vb + g.off, v0, sizeof(double) * g.n, cudaMemcpyDefault, st));
    SKS_TRY(halo_exchange(c, g, vb));
    SKS_TRY(first_column(c, b, 2, g.kind == SKS_OP_CSR ? vb + g.off : vb, nullptr));
  } else {  // unnormalised block basis: sigma = 1 for every column (B = W)
    SKS_CK(c, launch_eye_ones(nullptr, 0, 0, c->sigma.as<double>(), d + bs + 2, st));
    ++c->launches;
  }
  const uint64_t key = sks_key(o->seed, 0u);
  if (o->sketch != SKS_SKETCH_SPARSE && o->sketch != SKS_SKETCH_SRFT) return fail(c, SKS_EINVAL, "unknown sketch");
  if (o->sketch == SKS_SKETCH_SRFT && c->nranks > 1)
    return fail(c, SKS_EUNSUPPORTED, "the SRFT sketch is single-GPU (the DCT mixes all rows)");
  c->sketch_kind = o->sketch;
  c->sk_seed = o->seed;
  c->sk_cycle = 0;
  float t_basis_ms = 0.f;
  int qr_done = 0;  // columns of SB already factored during the basis loop (single-vector bases)
  const double bytes0 = b.bytes;
  if (blk)
    SKS_TRY(block_basis_and_sketch(c, b, v0, bs, d / bs, s, zeta, key, JB, &t_basis_ms));
  else
    SKS_TRY(basis_and_sketch(c, b, d, s, zeta, key, JB, true, &t_basis_ms, &qr_done));
  const double bytes_basis = b.bytes - bytes0;
  CtrlBlock* hc = c->h_ctrl;
  int de = d;
  int flags = 0;
  if (hc->stop_col < INT_MAX) {
    de = std::min(d, hc->stop_col);
    flags |= SKS_WARN_BREAKDOWN;
  }
  if (de < 2) return fail(c, SKS_EINVAL, "basis broke down before 2 columns");
  cudaEvent_t ev_s0 = c->ev_b0, ev_s1 = c->ev_b1;
  SKS_CK(c, cudaEventRecord(ev_s0, st));
  // ---- QR of SB[:, :de] (already done during the basis loop unless the basis broke down early)
  if (qr_done != de) {
    for (int j0 = 0; j0 < de; j0 += JB) {
      const int J = std::min(JB, de - j0);
      SKS_TRY(qr_append(c, b, 1, j0, J, s, 0, de, st));
    }
  }
  SKS_TRY(ensure(c, c->Mh, sizeof(double) * (size_t)de * de));
  SKS_TRY(ensure(c, c->Mh2, sizeof(double) * (size_t)de * de));
  if (!blk) {
    // ---- t = T^-1 U^T S w_de ; Mhat = Hbar[:de,:de] + t e_{de}^T
    SKS_CK(c, launch_form_cols(2, c->SW.as<double>(), s, de, 1, b.k, c->H.as<double>(), b.ldH,
                               c->sigma.as<double>(), c->gam.as<double>(), c->Xp.as<double>(), 1, 1, st));
    SKS_CK(c, launch_utx(c->U.as<double>(), s, s, de, c->Xp.as<double>(), 1, c->Zb.as<double>(), nullptr, 0, 0, 0,
                         c->bgsw.as<double>(), c->bgsc.as<int>(), st));
    SKS_CK(c, launch_trsv(c->T.as<double>(), b.ncol, de, c->Zb.as<double>(), nullptr, nullptr, c->coef.as<double>(),
                          st));
    SKS_CK(c, launch_build_mhat(c->H.as<double>(), b.ldH, de, c->coef.as<double>(), c->gam.as<double>(),
                                c->Mh.as<double>(), st));
  }
  SKS_CK(c, cudaEventRecord(c->ev_fork, st));
  SKS_CK(c, cudaStreamWaitEvent(c->side, c->ev_fork, 0));
  // ---- side stream, concurrent with the one-CTA eigen-solve: C = SB, D = SAB (for the sketched
  //      residual estimate) and kappa(T)
  SKS_TRY(ensure(c, c->SAB, sizeof(double) * (size_t)s * de));
  SKS_TRY(ensure(c, c->SB, sizeof(double) * (size_t)s * de));
  if (blk)  // S A B through the block recurrence from the sketched B_1..B_{p+1} (reading O34)
    SKS_CK(c, launch_block_sab(c->SW.as<double>(), s, bs, de / bs, b.sa.cheb_rho, b.sa.cheb_c, b.sa.cheb_e,
                               c->SAB.as<double>(), c->side));
  else
    SKS_CK(c, launch_form_cols(0, c->SW.as<double>(), s, 0, de, b.k, c->H.as<double>(), b.ldH,
                               c->sigma.as<double>(), c->gam.as<double>(), c->SAB.as<double>(), 1, s, c->side));
  SKS_CK(c, launch_form_cols(1, c->SW.as<double>(), s, 0, de, b.k, c->H.as<double>(), b.ldH, c->sigma.as<double>(),
                             c->gam.as<double>(),
                             c->SB.as<double>(), 1, s, c->side));
  SKS_CK(c, launch_cond(c->T.as<double>(), b.ncol, de, 12, nullptr, c->small.as<double>() + 8, c->side));
  SKS_CK(c, cudaEventRecord(c->ev_join, c->side));
  // ---- stabilised sRR (reading O33): truncated SVD SB = U Sigma V^T (one-sided Jacobi);
  //      the r x r problem M_r = Sigma_r^-1 U_r^T SAB V_r replaces Mhat, y = V_r z
  const double ctol = o->cond_tol > 0 ? o->cond_tol : 1e14;
  bool stab = o->stabilize == SKS_SRR_STABILIZE_ALWAYS;
  if (o->stabilize == SKS_SRR_STABILIZE_IF_ILL) {  // Alg. 2: test kappa_2(T) first
    SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));
    SKS_CK(c, cudaMemcpyAsync(c->h_small + 8, c->small.as<double>() + 8, sizeof(double), cudaMemcpyDeviceToHost, st));
    SKS_CK(c, cudaStreamSynchronize(st));
    stab = !(c->h_small[8] <= ctol);  // a non-finite estimate counts as ill-conditioned
  }
  int rr = de;  // order of the small eigenproblem
  if (stab) {
    SKS_TRY(ensure(c, c->svw, sizeof(double) * ((size_t)s * de + (size_t)de * de + de + 16)));
    SKS_TRY(ensure(c, c->svs, sizeof(double) * ((size_t)de + 64)));
    SKS_TRY(ensure(c, c->svU, sizeof(double) * (size_t)s * de));
    SKS_TRY(ensure(c, c->svV, sizeof(double) * (size_t)de * de));
    SKS_TRY(ensure(c, c->svH, sizeof(double) * (size_t)de * de));
    double* sig = c->svs.as<double>();
    int* svout = reinterpret_cast<int*>(sig + de + 8);
    SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));  // SB, SAB from the side stream
    SKS_CK(c, launch_jacobi_svd(c->SB.as<double>(), s, s, de, ctol, 60, c->svw.as<double>(), sig,
                                c->svU.as<double>(), c->svV.as<double>(), svout, st));
    int* hsv = reinterpret_cast<int*>(c->h_small + 16);
    SKS_CK(c, cudaMemcpyAsync(hsv, svout, sizeof(int) * 3, cudaMemcpyDeviceToHost, st));
    SKS_CK(c, cudaStreamSynchronize(st));
    rr = hsv[0];
    if (!hsv[2]) return fail(c, SKS_ENOTCONV, "Jacobi SVD of SB did not converge");
    if (rr < 2) return fail(c, SKS_EINVAL, "truncated rank of SB below 2");
    SKS_CK(c, launch_small_gemm(rr, de, s, c->svU.as<double>(), s, 1, c->SAB.as<double>(), s, 0, nullptr, 0,
                                c->svH.as<double>(), de, st));  // U_r^T SAB
    SKS_CK(c, launch_small_gemm(rr, rr, de, c->svH.as<double>(), de, 0, c->svV.as<double>(), de, 0, sig, 1,
                                c->Mh.as<double>(), rr, st));  // Sigma_r^-1 (U_r^T SAB) V_r
    // Hessenberg form for the eigen-solvers: M_r = Q H Q^T, V_r <- V_r Q (so y = V_r z_H)
    SKS_CK(c, launch_hess_reduce(c->Mh.as<double>(), rr, rr, c->svV.as<double>(), de, de,
                                 reinterpret_cast<unsigned*>(sig + de + 16), st));
    flags |= SKS_INFO_STABILIZED;
    c->launches += 4;
  }
  const bool useV = stab || blk;  // the eigenvectors z of the Hessenberg matrix map back through y = V z
  if (blk && !stab) {
    // Mhat = T^-1 (U^T SAB) (Eq. Mhat-form; dense for a block basis), then Q^T Mhat Q = H with
    // V = Q accumulated from the identity
    SKS_TRY(ensure(c, c->svs, sizeof(double) * ((size_t)de + 64)));
    SKS_TRY(ensure(c, c->svV, sizeof(double) * (size_t)de * de));
    SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));  // SAB from the side stream
    SKS_CK(c, launch_small_gemm(de, de, s, c->U.as<double>(), s, 1, c->SAB.as<double>(), s, 0, nullptr, 0,
                                c->Mh.as<double>(), de, st));  // U^T SAB
    SKS_CK(c, launch_trsm_upper(c->T.as<double>(), b.ncol, de, c->Mh.as<double>(), de, de, st));
    SKS_CK(c, launch_eye_ones(c->svV.as<double>(), de, de, nullptr, 0, st));
    SKS_CK(c, launch_hess_reduce(c->Mh.as<double>(), de, de, c->svV.as<double>(), de, de,
                                 reinterpret_cast<unsigned*>(c->svs.as<double>() + de + 16), st));
    c->launches += 4;
  }
  const int nev_e = std::min(nev, rr);
  SKS_CK(c, cudaMemcpyAsync(c->Mh2.p, c->Mh.p, sizeof(double) * (size_t)rr * rr, cudaMemcpyDeviceToDevice, st));
  SKS_TRY(ensure(c, c->wr, sizeof(double) * de));
  SKS_TRY(ensure(c, c->wi, sizeof(double) * de));
  SKS_TRY(ensure(c, c->sel, sizeof(int) * 64, true));
  SKS_TRY(ensure(c, c->th, sizeof(double) * 64));
  int* d_info = c->sel.as<int>() + 32;
  int* d_nsel = c->sel.as<int>() + 31;
  SKS_CK(c, cudaMemsetAsync(d_info, 0, sizeof(int) * 8, st));
  SKS_CK(c, launch_hqr(c->Mh2.as<double>(), rr, rr, c->wr.as<double>(), c->wi.as<double>(), d_info, st));
  double* th_re = c->th.as<double>();
  double* th_im = th_re + 32;
  SKS_CK(c, launch_select(c->wr.as<double>(), c->wi.as<double>(), rr, nev_e, c->sel.as<int>(), d_nsel, th_re, th_im,
                          st));
  SKS_TRY(ensure(c, c->ework, sizeof(double) * inverse_iteration_work_doubles(de, nmax)));
  SKS_TRY(ensure(c, c->yr, sizeof(double) * (size_t)de * nmax, true));
  SKS_TRY(ensure(c, c->yi, sizeof(double) * (size_t)de * nmax, true));
  SKS_CK(c, cudaMemsetAsync(c->yr.p, 0, sizeof(double) * (size_t)de * nmax, st));
  SKS_CK(c, cudaMemsetAsync(c->yi.p, 0, sizeof(double) * (size_t)de * nmax, st));
  SKS_CK(c, launch_inverse_iteration(c->Mh.as<double>(), rr, th_re, th_im, d_nsel, nmax, c->ework.as<double>(),
                                     c->yr.as<double>(), c->yi.as<double>(), 3, 0.0, st));
  SKS_CK(c, cudaStreamWaitEvent(st, c->ev_join, 0));
  const double* ys_r = c->yr.as<double>();
  const double* ys_i = c->yi.as<double>();
  if (useV) {  // y = V_r z (de x nmax)
    SKS_TRY(ensure(c, c->y2r, sizeof(double) * (size_t)de * nmax));
    SKS_TRY(ensure(c, c->y2i, sizeof(double) * (size_t)de * nmax));
    SKS_CK(c, launch_small_gemm(de, nmax, rr, c->svV.as<double>(), de, 0, c->yr.as<double>(), rr, 0, nullptr, 0,
                                c->y2r.as<double>(), de, st));
    SKS_CK(c, launch_small_gemm(de, nmax, rr, c->svV.as<double>(), de, 0, c->yi.as<double>(), rr, 0, nullptr, 0,
                                c->y2i.as<double>(), de, st));
    ys_r = c->y2r.as<double>();
    ys_i = c->y2i.as<double>();
    c->launches += 2;
  }
  double* d_rest = c->small.as<double>() + 128;
  SKS_CK(c, launch_srr_rest(c->SAB.as<double>(), c->SB.as<double>(), s, de, ys_r, ys_i,
                            th_re, th_im, d_nsel, nmax, d_rest, st));
  SKS_CK(c, cudaEventRecord(ev_s1, st));
  c->launches += 14;
  // ---- Ritz vectors x_i = B y_i and true residuals ||A x - theta x|| / ||x||
  SKS_TRY(ensure(c, c->Xr, sizeof(double) * (size_t)g.ld * nmax));
  SKS_TRY(ensure(c, c->Xi, sizeof(double) * (size_t)g.ld * nmax));
  // ghost planes must be zero (Dirichlet) for the residual stencil: clear the whole ghost layout
  // (the buffers may hold another geometry's data from an earlier call)
  SKS_CK(c, cudaMemsetAsync(c->Xr.p, 0, sizeof(double) * (size_t)g.ld * nmax, st));
  SKS_CK(c, cudaMemsetAsync(c->Xi.p, 0, sizeof(double) * (size_t)g.ld * nmax, st));
  SKS_TRY(ensure(c, c->rcoef, sizeof(double) * ritz_coef_doubles(de)));
  SKS_CK(c, launch_ritz_vectors(c->W.as<double>(), g.ld, g.off, g.n, de, c->sigma.as<double>(), ys_r,
                                ys_i, de, th_re, th_im, d_nsel, nmax, c->rcoef.as<double>(),
                                c->Xr.as<double>(), c->Xi.as<double>(), g.ld, g.off, c->num_sms, st));
  c->launches += 2;
  const int rgrid = c->num_sms * 2;
  double* rpart = c->tmp.as<double>();
  SKS_TRY(ensure(c, c->tmp, sizeof(double) * (size_t)rgrid * nmax * 2 + 64));
  rpart = c->tmp.as<double>();
  if (g.kind != SKS_OP_CSR) {
    for (int v = 0; v < nmax; ++v) {
      SKS_TRY(halo_exchange(c, g, c->Xr.as<double>() + (int64_t)v * g.ld));
      SKS_TRY(halo_exchange(c, g, c->Xi.as<double>() + (int64_t)v * g.ld));
    }
    SKS_CK(c, launch_ritz_residual_stencil(g.dim, g.m, g.nz, g.plane, g.off, g.ld, g.cc, g.cm, g.cp, nmax,
                                           c->Xr.as<double>(), c->Xi.as<double>(), th_re, th_im, rpart, rgrid, st));
    ++c->launches;
  } else {
    SKS_TRY(ensure(c, c->AXr, sizeof(double) * (size_t)g.ld * nmax));
    SKS_TRY(ensure(c, c->AXi, sizeof(double) * (size_t)g.ld * nmax));
    for (int v = 0; v < nmax; ++v) {
      for (int part = 0; part < 2; ++part) {
        const double* src = (part ? c->Xi : c->Xr).as<double>() + (int64_t)v * g.ld;
        double* dst = (part ? c->AXi : c->AXr).as<double>() + (int64_t)v * g.ld;
        const double* xg = nullptr;
        SKS_TRY(csr_gather(c, g, src, &xg, b.maxn));
        SKS_CK(c, launch_csr_spmv(g.n, b.rp, b.ci, b.va, xg, dst, nullptr, 0, nullptr, 0, 0, 0, k,
                                  c->part2.as<double>(), b.step_grid, st, nullptr, b.ell_ci, b.ell_va, b.ell_w));
        ++c->launches;
      }
    }
    SKS_CK(c, launch_complex_residual(g.n, c->AXr.as<double>(), c->AXi.as<double>(), c->Xr.as<double>(),
                                      c->Xi.as<double>(), g.ld, g.ld, nmax, th_re, th_im, rpart, rgrid, st));
    ++c->launches;
  }
  double* rsum = c->small.as<double>() + 256;
  SKS_CK(c, launch_sum_partials(rpart, rgrid, nmax * 2, nmax * 2, rsum, st));
  ++c->launches;
  SKS_TRY(allreduce_sum(c, rsum, (size_t)nmax * 2, st));
  SKS_CK(c, cudaEventRecord(c->ev_t1, st));
  // ---- outputs
  double* hs = c->h_small;
  SKS_CK(c, cudaMemcpyAsync(hs, c->small.p, sizeof(double) * 512, cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaMemcpyAsync(hs + 512, c->th.p, sizeof(double) * 64, cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaMemcpyAsync(hs + 576, c->sel.p, sizeof(int) * 64, cudaMemcpyDeviceToHost, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  SKS_CK(c, cudaGetLastError());
  const int* hsel = reinterpret_cast<const int*>(hs + 576);
  const int nsel = hsel[31];
  const int hinfo = hsel[32];
  if (getenv("SKS_DEBUG_HQR")) fprintf(stderr, "hqr: d=%d sweeps=%d bulge_steps=%d chase_kcyc=%d total_kcyc=%d "
                                       "(HQ_PROF: setup %d trans %d last %d)\n", de, hsel[33], hsel[34], hsel[35],
                                       hsel[36], hsel[37], hsel[38], hsel[39]);
  if (hinfo != 0) return fail(c, SKS_ENOTCONV, "QR algorithm did not converge on Mhat");
  if (getenv("SKS_DEBUG_SRR") && stab) fprintf(stderr, "srr stabilised: rank %d of %d\n", rr, de);
  for (int v = 0; v < nsel; ++v) {
    theta_re[v] = hs[512 + v];
    theta_im[v] = hs[512 + 32 + v];
    if (res_est) res_est[v] = hs[128 + v];
    if (res_true) res_true[v] = std::sqrt(hs[256 + 2 * v] / hs[256 + 2 * v + 1]);
  }
  if (X_re && X_im) {
    for (int v = 0; v < nsel; ++v) {
      SKS_CK(c, cudaMemcpyAsync(X_re + (int64_t)v * g.n, c->Xr.as<double>() + (int64_t)v * g.ld + g.off,
                                sizeof(double) * g.n, cudaMemcpyDefault, st));
      SKS_CK(c, cudaMemcpyAsync(X_im + (int64_t)v * g.n, c->Xi.as<double>() + (int64_t)v * g.ld + g.off,
                                sizeof(double) * g.n, cudaMemcpyDefault, st));
    }
    SKS_CK(c, cudaStreamSynchronize(st));
  }
  if (info) {
    memset(info, 0, sizeof(*info));
    info->columns = de;
    info->flags = flags | (hs[8] > (o->cond_tol > 0 ? o->cond_tol : 1e14) ? SKS_WARN_COND : 0);
    info->nev_out = nsel;
    info->rank = rr;
    info->cond_SB = hs[8];
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->ev_t0, c->ev_t1);
    info->t_total_s = ms * 1e-3;
    info->t_basis_s = t_basis_ms * 1e-3;
    cudaEventElapsedTime(&ms, ev_s0, ev_s1);
    info->t_small_s = ms * 1e-3;
    info->bytes_basis = bytes_basis;
    info->kernel_launches = c->launches - launches0;
    info->steps = b.steps;
  }
  return SKS_OK;
}

// ------------------------------------------------------------------------------------
// test / parity entry points
// ------------------------------------------------------------------------------------
extern "C" sks_status sks_sketch_apply(sks_ctx* c, int64_t n_global, int64_t row_begin, int64_t row_end, int32_t s,
                                       int32_t zeta, uint64_t seed, uint32_t cycle, const double* M, int64_t ldm,
                                       int32_t cc, double* SM) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  const int64_t n = row_end - row_begin;
  if (!M || !SM || n <= 0 || row_begin < 0 || row_end > n_global || cc < 1 || ldm < n || s < 1 || s > SKS_SMAX ||
      zeta < 1 || zeta > std::min<int>(s, SKS_ZETA_MAX))
    return fail(c, SKS_EINVAL, "bad sketch_apply arguments");
  cudaSetDevice(c->device);
  cudaStream_t st = c->main();
  const int64_t ldd = (n + 1) / 2 * 2;
  SKS_TRY(ensure(c, c->tmp, sizeof(double) * (size_t)ldd * cc));
  SKS_TRY(ensure(c, c->SAB, sizeof(double) * (size_t)s * cc));
  const int grid = sketch_grid(c->num_sms, n);
  SKS_TRY(ensure(c, c->partsk, sizeof(double) * sketch_part_doubles(grid, SKS_JB, s)));
  SKS_CK(c, cudaMemcpy2DAsync(c->tmp.p, sizeof(double) * ldd, M, sizeof(double) * ldm, sizeof(double) * n, cc,
                              cudaMemcpyDefault, st));
  const uint64_t key = sks_key(seed, cycle);
  c->sketch_kind = SKS_SKETCH_SPARSE;
  Geo gq;
  gq.n = n;
  gq.row_begin = row_begin;
  const void* plan = nullptr;
  SKS_TRY(sketch_plan(c, gq, s, zeta, key, st, &plan));
  for (int c0 = 0; c0 < cc; c0 += SKS_JB) {
    const int J = std::min(SKS_JB, cc - c0);
    SKS_CK(c, launch_sketch(c->tmp.as<double>() + (int64_t)c0 * ldd, ldd, n, row_begin, J, s, zeta, key,
                            c->partsk.as<double>(), grid, c->SAB.as<double>() + (int64_t)c0 * s, s, 0, st,
                            &c->launches, plan));
  }
  SKS_TRY(allreduce_sum(c, c->SAB.as<double>(), (size_t)s * cc, st));
  SKS_CK(c, cudaMemcpyAsync(SM, c->SAB.p, sizeof(double) * (size_t)s * cc, cudaMemcpyDefault, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  return SKS_OK;
}

extern "C" sks_status sks_srft_apply(sks_ctx* c, int64_t n, int32_t s, uint64_t seed, uint32_t cycle,
                                     const double* M, int32_t cc, double* SM) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  if (!M || !SM || n < 1 || s < 1 || s > n || s > SKS_SMAX || cc < 1 || n >= (int64_t(1) << 31))
    return fail(c, SKS_EINVAL, "bad srft_apply arguments");
  if (c->nranks > 1) return fail(c, SKS_EUNSUPPORTED, "the SRFT sketch is single-GPU");
  cudaSetDevice(c->device);
  cudaStream_t st = c->main();
  SKS_TRY(ensure(c, c->tmp, sizeof(double) * (size_t)n * cc));
  SKS_TRY(ensure(c, c->SAB, sizeof(double) * (size_t)s * cc));
  SKS_TRY(ensure(c, c->srft_w, sizeof(double) * srft_work_doubles(n, SKS_JB)));
  SKS_CK(c, cudaMemcpyAsync(c->tmp.p, M, sizeof(double) * (size_t)n * cc, cudaMemcpyDefault, st));
  c->sketch_kind = SKS_SKETCH_SRFT;
  c->sk_seed = seed;
  c->sk_cycle = cycle;
  Geo gq;
  gq.n = n;
  gq.row_begin = 0;
  const void* plan = nullptr;
  SKS_TRY(sketch_plan(c, gq, s, 8, 0, st, &plan));
  const uint64_t key = srft_key_host(seed, cycle);
  for (int c0 = 0; c0 < cc; c0 += SKS_JB) {
    const int J = std::min(SKS_JB, cc - c0);
    SKS_CK(c, launch_srft(c->tmp.as<double>() + (int64_t)c0 * n, n, n, J, s, key, c->srft_q.as<int32_t>(),
                          c->srft_w.as<double>(), &c->srft_cache, c->SAB.as<double>() + (int64_t)c0 * s, s,
                          c->num_sms, st));
  }
  SKS_CK(c, cudaMemcpyAsync(SM, c->SAB.p, sizeof(double) * (size_t)s * cc, cudaMemcpyDefault, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  return SKS_OK;
}

extern "C" sks_status sks_sketch_table(sks_ctx* c, int64_t row_begin, int64_t count, int32_t s, int32_t zeta,
                                       uint64_t seed, uint32_t cycle, int32_t* q, int8_t* sign) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  if (!q || !sign || count < 0 || s < 1 || zeta < 1 || zeta > std::min<int>(s, SKS_ZETA_MAX))
    return fail(c, SKS_EINVAL, "bad sketch_table arguments");
  if (count == 0) return SKS_OK;
  cudaSetDevice(c->device);
  cudaStream_t st = c->main();
  SKS_TRY(ensure(c, c->cig, sizeof(int32_t) * (size_t)count * zeta));
  SKS_TRY(ensure(c, c->tmp, sizeof(int8_t) * (size_t)count * zeta));
  SKS_CK(c, launch_sketch_table(row_begin, count, s, zeta, sks_key(seed, cycle), c->cig.as<int32_t>(),
                                c->tmp.as<int8_t>(), st));
  SKS_CK(c, cudaMemcpyAsync(q, c->cig.p, sizeof(int32_t) * (size_t)count * zeta, cudaMemcpyDefault, st));
  SKS_CK(c, cudaMemcpyAsync(sign, c->tmp.p, sizeof(int8_t) * (size_t)count * zeta, cudaMemcpyDefault, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  return SKS_OK;
}

extern "C" sks_status sks_apply_operator(sks_ctx* c, const sks_operator* A, const double* x, double* y) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  if (!A || !x || !y) return fail(c, SKS_EINVAL, "NULL argument");
  cudaSetDevice(c->device);
  cudaStream_t st = c->main();
  Basis b;
  SKS_TRY(setup_basis(c, A, 2, 2, &b));
  const Geo& g = b.g;
  double* xb = c->xb.as<double>();
  double* yb = c->vb.as<double>();
  SKS_CK(c, cudaMemsetAsync(xb, 0, sizeof(double) * g.ld, st));
  SKS_CK(c, cudaMemcpyAsync(xb + g.off, x, sizeof(double) * g.n, cudaMemcpyDefault, st));
  if (g.kind != SKS_OP_CSR) {
    SKS_TRY(halo_exchange(c, g, xb));
    SKS_CK(c, launch_apply_stencil(g.dim, g.m, g.nz, g.plane, g.off, g.cc, g.cm, g.cp, xb, yb, c->num_sms, st));
  } else {
    const double* xg = nullptr;
    SKS_TRY(csr_gather(c, g, xb, &xg, b.maxn));
    SKS_CK(c, launch_csr_spmv(g.n, b.rp, b.ci, b.va, xg, yb, nullptr, 0, nullptr, 0, 0, 0, 2, c->part2.as<double>(),
                              b.step_grid, st, nullptr, b.ell_ci, b.ell_va, b.ell_w));
  }
  ++c->launches;
  SKS_CK(c, cudaMemcpyAsync(y, yb + g.off, sizeof(double) * g.n, cudaMemcpyDefault, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  return SKS_OK;
}

extern "C" sks_status sks_basis(sks_ctx* c, const sks_operator* A, const double* r0, int32_t k, int32_t ncols,
                                double* B_out, double* H_out) {
  if (!c) return SKS_EINVAL;
  c->err.clear();
  if (!A || !r0 || !B_out || ncols < 1 || k < 1 || k > SKS_KMAX) return fail(c, SKS_EINVAL, "bad sks_basis arguments");
  cudaSetDevice(c->device);
  cudaStream_t st = c->main();
  Basis b;
  SKS_TRY(setup_basis(c, A, k, ncols + 2, &b));
  const Geo& g = b.g;
  SKS_TRY(ensure(c, c->tmp, sizeof(double) * (size_t)std::max<int64_t>(g.n * ncols, 4096)));
  double* vb = c->vb.as<double>();
  SKS_CK(c, cudaMemsetAsync(vb, 0, sizeof(double) * g.ld, st));
  SKS_CK(c, cudaMemcpyAsync(vb + g.off, r0, sizeof(double) * g.n, cudaMemcpyDefault, st));
  SKS_TRY(halo_exchange(c, g, vb));
  SKS_CK(c, launch_ctrl_reset(c->ctrl.as<CtrlBlock>(), -1.0, 0.0, st));
  ++c->launches;
  SKS_TRY(first_column(c, b, 2, g.kind == SKS_OP_CSR ? vb + g.off : vb, nullptr));
  SKS_TRY(basis_and_sketch(c, b, ncols, 0, 0, 0, SKS_JB, false, nullptr));
  SKS_CK(c, launch_scale_cols(c->W.as<double>(), g.ld, g.off, g.n, ncols, c->sigma.as<double>(), c->tmp.as<double>(),
                              g.n, st));
  ++c->launches;
  SKS_CK(c, cudaMemcpyAsync(B_out, c->tmp.p, sizeof(double) * (size_t)g.n * ncols, cudaMemcpyDefault, st));
  if (H_out && ncols >= 2)
    SKS_CK(c, cudaMemcpy2DAsync(H_out, sizeof(double) * ncols, c->H.p, sizeof(double) * b.ldH,
                                sizeof(double) * ncols, ncols - 1, cudaMemcpyDefault, st));
  SKS_CK(c, cudaStreamSynchronize(st));
  if (c->h_ctrl->stop_col < ncols) {
    c->err = "breakdown at column " + std::to_string(c->h_ctrl->stop_col);
    return SKS_OK;  // columns past the breakdown are not meaningful (flagged via sks_last_error)
  }
  return SKS_OK;
}
