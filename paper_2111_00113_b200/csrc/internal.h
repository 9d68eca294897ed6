// internal.h -- host-side launchers shared between the kernel files and the driver.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <algorithm>

struct StepArgs;
struct CtrlBlock;

namespace sks {

// stencil.cu
int step_km(int k);
cudaError_t launch_step_stencil(const StepArgs& a, int grid, cudaStream_t st);
void stencil_tiling(int dim, int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid);
cudaError_t launch_apply_stencil(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off, double cc, double cm,
                                 double cp, const double* x, double* y, int num_sms, cudaStream_t st);
cudaError_t launch_ritz_residual_stencil(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off, int64_t ld,
                                         double cc, double cm, double cp, int nvec, const double* Xr,
                                         const double* Xi, const double* thr, const double* thi, double* partials,
                                         int grid, cudaStream_t st);

// stencil_tma.cu (even m: TMA-fed persistent kernels)
bool stencil_tma_supported(int dim, int64_t m, int k);
void stencil_tma_tiling(int dim, int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid);
cudaError_t launch_step_stencil_tma(const StepArgs& a, const double* W, int64_t ncol, const double* xb,
                                    const double* fb, const double* vb, int grid, cudaStream_t st, void** cache);
void stencil_tma_free(void* cache);

// stencil_zm.cu (3D, even m: TMA-fed z-march kernel)
bool stencil_zm_supported(int dim, int64_t m, int k);
void stencil_zm_tiling(int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid);
cudaError_t launch_step_stencil_zm(const StepArgs& a, const double* W, int64_t ncol, const double* xb,
                                   const double* fb, const double* vb, int grid, cudaStream_t st, void** cache);
void stencil_zm_free(void* cache);

// stencil_coop.cu (small problems: a batch of columns in one cooperative launch, single rank)
int coop_grid(int main_sms);
int coop1_lines(int dim, int64_t m, int64_t nz, int k, int max_grid);
cudaError_t launch_step_coop1(const StepArgs& a, int j0, int j1, int grid_prev0, double* part, int pstride,
                              unsigned* sync, int lines, cudaStream_t st);
cudaError_t launch_step_coop(const StepArgs& a, int j0, int j1, int grid_prev0, double* part, int pstride,
                             unsigned* sync, int grid, cudaStream_t st);
cudaError_t launch_ctrl_copy(CtrlBlock* dst, const CtrlBlock* src, cudaStream_t st);
cudaError_t launch_ctrl_merge(CtrlBlock* real, const CtrlBlock* priv, int first, cudaStream_t st);

// stencil_ym.cu (2D, even m: TMA-fed y-march kernel)
bool stencil_ym_supported(int dim, int64_t m, int k);
void stencil_ym_tiling(int64_t m, int64_t nz, int num_sms, StepArgs* a, int* grid);
cudaError_t launch_step_stencil_ym(const StepArgs& a, const double* W, int64_t ncol, const double* xb,
                                   const double* fb, const double* vb, int grid, cudaStream_t st, void** cache);
void stencil_ym_free(void* cache);

// srft.cu (SRFT sketch, reading O32)
uint64_t srft_key_host(uint64_t seed, uint32_t cycle);
void srft_rows_host(int64_t n, int s, uint64_t key, int32_t* q);
size_t srft_work_doubles(int64_t n, int J);
cudaError_t launch_srft(const double* M, int64_t ldm, int64_t n, int J, int s, uint64_t key, const int32_t* q,
                        double* work, void** cache, double* out, int64_t ldo, int num_sms, cudaStream_t st);
void srft_free(void* cache);

// sketch.cu
int sketch_grid(int num_sms, int64_t nrows);
size_t sketch_part_doubles(int grid, int J, int s);
// plan: per-cycle sketch plan of these rows (launch_sketch_plan), or NULL for the generic kernel
cudaError_t launch_sketch(const double* M, int64_t ldm, int64_t nrows, int64_t row_begin, int J, int s, int zeta,
                          uint64_t key, double* part, int grid, double* out, int64_t ldo, int accumulate,
                          cudaStream_t st, int64_t* launches, const void* plan);
bool sketch_plan_supported(int s, int zeta);
size_t sketch_plan_bytes(int64_t nrows, int s, int zeta);
cudaError_t launch_sketch_plan(int64_t nrows, int64_t row_begin, int s, int zeta, uint64_t key, void* plan,
                               int num_sms, cudaStream_t st);
cudaError_t launch_sketch_table(int64_t row_begin, int64_t count, int s, int zeta, uint64_t key, int32_t* q,
                                int8_t* sign, cudaStream_t st);

// smallside.cu
cudaError_t launch_form_cols(int mode, const double* SW, int s, int j0, int J, int k, const double* H, int ldH,
                             const double* sigma, const double* gam, double* X, int64_t ldq, int64_t ldj,
                             cudaStream_t st);
cudaError_t launch_utx(const double* U, int ldu, int s, int j0, const double* X, int J, double* Z, double* T,
                       int ldT, int tc0, int tacc, double* ws, int* cnt, cudaStream_t st);
cudaError_t launch_xmuz(const double* U, int ldu, int s, int j0, double* X, int J, const double* Z, double* ws,
                        int* cnt, cudaStream_t st);
size_t bgs_workspace_doubles(int s, int ncol);
size_t panel_smem(int s, int J);
cudaError_t launch_panel(double* X, int s, int J, int j0, double* U, int ldu, double* T, int ldT, double* rvec,
                         double* rho, double* rest, CtrlBlock* ctrl, int track_res, int max_cols,
                         cudaStream_t st);
cudaError_t launch_trsv(const double* T, int ldT, int n, const double* b, const double* scale, double* yout,
                        double* out, cudaStream_t st);
cudaError_t launch_cond(const double* T, int ldT, int n, int iters, CtrlBlock* ctrl, double* out,
                        cudaStream_t st);
cudaError_t launch_assemble(double* x, const double* W, int64_t ld, int64_t off, int64_t n, const double* coef,
                            const int* ncp, int nc_max, int num_sms, cudaStream_t st);
size_t ritz_coef_doubles(int nc);
// Ritz vectors X_v = W diag(sigma) y_v for the nsel selected v (conjugate partners and real y
// share compact columns); work: ritz_coef_doubles(nc) doubles.  Xr/Xi must be zero on entry.
cudaError_t launch_ritz_vectors(const double* W, int64_t ld, int64_t off, int64_t n, int nc, const double* sigma,
                                const double* yr, const double* yi, int ldy, const double* th_re,
                                const double* th_im, const int* nsel, int nmax, double* work, double* Xr,
                                double* Xi, int64_t ldx, int64_t xoff, int num_sms, cudaStream_t st);
cudaError_t launch_scale_cols(const double* W, int64_t ld, int64_t off, int64_t n, int nc, const double* sigma,
                              double* out, int64_t ldo, cudaStream_t st);
cudaError_t launch_complex_residual(int64_t n, const double* Axr, const double* Axi, const double* xr,
                                    const double* xi, int64_t ldx, int64_t ldax, int nvec, const double* thr,
                                    const double* thi, double* partials, int grid, cudaStream_t st);
cudaError_t launch_sum_partials(const double* part, int grid, int stride, int ncomp, double* out, cudaStream_t st);
cudaError_t launch_ctrl_reset(CtrlBlock* c, double thr, double fnorm, cudaStream_t st);
cudaError_t launch_remap_cols(int64_t nnz, const int32_t* ci_global, int32_t* ci_out, int nranks,
                              const int64_t* rb_dev, int64_t maxn, cudaStream_t st);

// eig.cu
cudaError_t launch_build_mhat(const double* H, int ldH, int d, const double* t, const double* gam, double* Mh,
                              cudaStream_t st);
cudaError_t launch_hqr(double* a, int n, int lda, double* wr, double* wi, int* info, cudaStream_t st);
cudaError_t launch_select(const double* wr, const double* wi, int n, int nev, int* sel, int* nsel, double* th_re,
                          double* th_im, cudaStream_t st);
size_t inverse_iteration_work_doubles(int d, int nmax);
cudaError_t launch_inverse_iteration(const double* Mh, int d, const double* th_re, const double* th_im,
                                     const int* nsel, int nmax, double* work, double* yr, double* yi, int iters,
                                     double anorm, cudaStream_t st);
// stencil_zm.cu: step-balanced partition of (tile, plane|line) units over `grid` CTAs (ub[grid+1])
bool step_partition(int64_t units, int64_t nz, int grid, int zs, int maxg, int32_t* ub);
// svd.cu: stabilised sRR (reading O33)
cudaError_t launch_jacobi_svd(const double* M, int ldm, int rows, int n, double tol, int max_sweeps, double* work,
                              double* sigma, double* Ut, double* Vs, int* out, cudaStream_t st);
cudaError_t launch_hess_reduce(double* M, int n, int ldm, double* V, int vrows, int ldv, unsigned* scratch,
                               cudaStream_t st);
cudaError_t launch_small_gemm(int M, int N, int K, const double* A, int lda, int ta, const double* B, int ldb,
                              int tb, const double* rs, int rs_inv, double* C, int ldc, cudaStream_t st);
cudaError_t launch_srr_rest(const double* D, const double* C, int s, int d, const double* yr, const double* yi,
                            const double* th_re, const double* th_im, const int* nsel, int nmax, double* rest,
                            cudaStream_t st);

// block.cu (block Chebyshev sRR)
cudaError_t launch_block_cheb(int dim, int64_t m, int64_t nz, int64_t plane, int64_t off, int64_t ld, double cc,
                              double cm, double cp, const double* in1, const double* in2, double* out, int ncols,
                              double alpha, double shift, double gamma, cudaStream_t st);
cudaError_t launch_block_sab(const double* SW, int s, int b, int p, double rho, double c, double e, double* SAB,
                             cudaStream_t st);
cudaError_t launch_trsm_upper(const double* T, int ldT, int n, double* X, int ldx, int nrhs, cudaStream_t st);
cudaError_t launch_eye_ones(double* V, int n, int ldv, double* sigma, int nc, cudaStream_t st);
cudaError_t launch_whiten_gemm(const double* W, int64_t ld, int64_t off, int64_t n, int J, const double* Z, int ldz,
                               double* Wn, double* part, int ngroups, cudaStream_t st);
cudaError_t launch_resid_restore(double* r, const double* g, const double* U, int ldu, const double* rho, int J, int s,
                                 cudaStream_t st);
cudaError_t launch_colsum(const double* part, int ng, int J, double* sums, cudaStream_t st);
cudaError_t launch_whiten_finish(const double* sums, int J, double* sigma, double* T, int ldT, CtrlBlock* ctrl,
                                 cudaStream_t st);
cudaError_t launch_scale_rows(double* Z, int J, int ldz, const double* sigma, cudaStream_t st);
cudaError_t launch_whiten_partials(const double* u, const double* const* v, const int* slot, int nv, int64_t n,
                                   int64_t plane, int64_t m, int dim, double cc, double cm, double cp, double* part,
                                   int grid, cudaStream_t st);
size_t mpk2d_smem(int64_t m, int64_t nz, int grid, int S);
cudaError_t launch_cheb_mpk2d(double* W, int64_t ld, int64_t off, int64_t m, int64_t nz, int64_t z0, int64_t mglob,
                              double cc, double cm, double cp, double rho, double c0, double e, int j, int S,
                              double* partc, int pstride, int zero_to, const CtrlBlock* ctrl, int grid,
                              cudaStream_t st);
cudaError_t launch_cheb_colsum(const double* part, int grid, int pstride, int j0, int j1, double* sums,
                               cudaStream_t st);
cudaError_t launch_cheb_finalize(const double* sums, int j0, int j1, double rho, double c0, double e, double* sigma,
                                 double* H, int ldH, double* mnorm, double* gam, CtrlBlock* ctrl, cudaStream_t st);

// csr.cu
cudaError_t launch_csr_spmv(int64_t n, const int32_t* rp, const int32_t* ci, const double* va, const double* xg,
                            double* out, const double* f, int mode, const double* W, int64_t ld, int lo, int nw,
                            int k, double* partials, int grid, cudaStream_t st, const CtrlBlock* ctrl = nullptr,
                            const int32_t* ell_ci = nullptr, const double* ell_va = nullptr, int ell_w = 0);
// ELL copy of a CSR matrix (column-major [ell_w][n], rows padded with (0, 0.0)); width = max row length
cudaError_t launch_csr_max_row(int64_t n, const int32_t* rp, int* out, cudaStream_t st);
cudaError_t launch_csr_to_ell(int64_t n, const int32_t* rp, const int32_t* ci, const double* va, int w, int32_t* eci,
                              double* eva, cudaStream_t st);
cudaError_t launch_csr_orth(int64_t n, int j, int k, double* W, int64_t ld, const double* mr, const double* pnorm,
                            int grid_n, const double* pdot, int grid_s, double* partials, double* sigma, double* H,
                            int ldH, double* mnorm, CtrlBlock* ctrl, int grid, cudaStream_t st);
cudaError_t launch_copy_norm(int64_t n, const double* src, double* dst, double* partials, int grid,
                             cudaStream_t st);

}  // namespace sks
