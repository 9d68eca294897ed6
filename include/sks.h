/*
 * sks.h -- C-ABI of the B200-native sketched-Krylov library (libsks.so).
 *
 * Hot path of sketched GMRES and sketched Rayleigh-Ritz, arXiv 2111.00113
 * (PAPER.md, cited as P:<line>):
 *   - Krylov basis by k-truncated Arnoldi, Eq. (partorth), Alg. 1 P:1296-1307;
 *   - sparse sign embedding S, Eq. (sparse-map) P:647-659;
 *   - sGMRES: SAB = UT, yhat = T^-1 U^T S r0, r_est = ||(I-UU^T) S r0||,
 *     x = x0 + B yhat (Eqs. sgmres-yhat/-rhat P:785-798; iterative form P:1351-1385;
 *     restarts P:938-957);
 *   - sRR: SB = UT, Mhat = T^-1 U^T SAB, eig(Mhat), r_est (Eqs. Mhat-form P:1598-1601,
 *     srr-resid-est P:1555-1559; Alg. 2).
 *
 * Conventions
 *   - All floating point is IEEE fp64.  All indices are 0-based.
 *   - Every pointer argument may be a HOST or a DEVICE (CUDA) pointer; the library
 *     detects which with cudaPointerGetAttributes and copies as needed.  Device
 *     pointers must live on the context's device.
 *   - The caller owns every buffer it passes in or out.  The library owns its
 *     device workspaces (inside sks_ctx; freed by sks_destroy).
 *   - No exception crosses this ABI.  Every call returns an sks_status; on error
 *     sks_last_error(ctx) holds a one-line message.  Numerical warnings (kappa(T) >
 *     cond_tol, breakdown) are reported in info->flags, never as an error.
 *   - Multi-GPU: one process per GPU.  Every rank calls each function collectively
 *     with its own contiguous row block [row_begin, row_end) (see sks_partition).
 *     Small-side outputs (theta, residuals, info) are identical on every rank.
 *   - No CPU fallback: if no CUDA device is usable, calls fail with SKS_ECUDA.
 */
#ifndef SKS_H
#define SKS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKS_ABI_VERSION 8

typedef enum {
  SKS_OK = 0,
  SKS_EINVAL = -1,       /* bad argument: sizes, kinds, non-finite input, NULL */
  SKS_ECUDA = -2,        /* CUDA runtime error (message in sks_last_error) */
  SKS_ENCCL = -3,        /* NCCL error */
  SKS_ENOMEM = -4,       /* device allocation failed */
  SKS_ENOTCONV = -5,     /* sgmres: tol not met within max_cycles; x is still the last iterate */
  SKS_EUNSUPPORTED = -6  /* valid request outside what this build implements */
} sks_status;

/* info->flags bits (warnings, never errors) */
enum {
  SKS_WARN_COND = 1,       /* kappa_2(T) > cond_tol (Alg. 1, Alg. 2) */
  SKS_WARN_BREAKDOWN = 2,  /* ||w_j|| <= 1e-14 ||m_{j-1}||: basis stopped early (reading O10) */
  SKS_WARN_STAGNATION = 4, /* reserved */
  SKS_INFO_ADAPTIVE_RESTART = 8, /* SKS_OPT_ADAPTIVE_RESTART ended at least one cycle early */
  SKS_INFO_STABILIZED = 16, /* sRR solved the truncated-SVD pencil (SKS_SRR_STABILIZE_*, reading O33) */
  SKS_INFO_WHITEN = 32      /* SKS_OPT_WHITEN whitened the basis at least once */
};

typedef struct sks_ctx sks_ctx;

/* ---- context ---------------------------------------------------------------- */

/* NCCL unique id (128 bytes) for a multi-rank context; call on rank 0 and
 * broadcast the bytes (e.g. torch.distributed.broadcast).  No GPU needed. */
sks_status sks_get_unique_id(unsigned char id[128]);

/* Create a context on CUDA device `device`.  nranks == 1: id may be NULL.
 * nranks > 1: collective over all ranks; creates an NCCL communicator. */
sks_status sks_create(sks_ctx** ctx, int device, int rank, int nranks,
                      const unsigned char* id);
sks_status sks_destroy(sks_ctx* ctx);

/* Single-process LOOPBACK transport (multi-rank testing with fewer GPUs than ranks): nranks
 * contexts in ONE process, one host thread per rank, all on one device, exchange their halos, all-reductions and
 * all-gathers by device-to-device copies ordered with CUDA events and host barriers instead of NCCL (the
 * library's own partition, ghost-plane and replicated-small-side code runs unchanged).  Every rank must call the
 * same entry points in the same order from its own thread, as with NCCL.  The group is owned by the caller:
 * create it once (nranks <= 16), create one context per rank with sks_create_loopback, destroy every context
 * before the group.  Errors: SKS_EINVAL (NULL, nranks out of range), SKS_ENOMEM, SKS_ECUDA. */
typedef struct sks_loopback sks_loopback;
sks_status sks_loopback_create(int nranks, sks_loopback** group);
sks_status sks_loopback_destroy(sks_loopback* group);
sks_status sks_create_loopback(sks_ctx** ctx, int device, int rank, sks_loopback* group);
const char* sks_last_error(const sks_ctx* ctx);   /* never NULL */
int sks_abi_version(void);

/* Launch the main (basis) work on `stream` (a cudaStream_t, e.g. torch's current
 * stream); NULL restores the library's own stream.  The small-side work runs on an
 * internal second stream that forks from and joins back into it, so events
 * recorded on `stream` bracket a whole call. */
sks_status sks_set_stream(sks_ctx* ctx, void* stream);

/* Row partition used by all entry points: contiguous blocks; stencils split
 * whole y-lines (2D) / z-planes (3D) as evenly as possible, CSR splits rows.
 * No GPU needed. */
sks_status sks_partition(int kind, int64_t m, int64_t n_global, int nranks, int rank,
                         int64_t* row_begin, int64_t* row_end);

/* ---- operator A ("access the matrix via products x -> Ax") --------- */

typedef enum {
  SKS_OP_STENCIL2D = 1,  /* 5-point -Lap(u) + beta (u_x + u_y), m x m interior grid */
  SKS_OP_STENCIL3D = 2,  /* 7-point -Lap(u) + beta (u_x + u_y + u_z), m^3 grid */
  SKS_OP_CSR = 3         /* general sparse matrix, CSR */
} sks_op_kind;

/* Stencils (reading O18): h = 1/(m+1), homogeneous Dirichlet, centred differences,
 * unscaled; row r = i + m*j (+ m^2*l), x fastest.  Coefficients: centre 2*dim/h^2,
 * "minus" neighbours (i-1, j-1, l-1) -1/h^2 - beta/(2h), "plus" -1/h^2 + beta/(2h).
 * CSR: rows [row_begin,row_end) of A; row_ptr has (row_end-row_begin+1) int32
 * entries starting at 0; col_idx are GLOBAL int32 column indices; val fp64.
 * The library copies the CSR arrays to the device once per call.  When the rows are near-uniform (longest row
 * w <= 32 and <= 1.25 x the average + 1) it also builds a column-major ELL copy (w x rows, 12 bytes per entry,
 * library-owned device memory reused across calls) that the SpMV reads instead; SKS_CSR_ELL=0 disables it. */
typedef struct {
  int32_t kind;            /* sks_op_kind */
  int32_t reserved0;
  int64_t m;               /* stencil: points per side (n_global = m^2 or m^3) */
  double beta;             /* stencil: convection coefficient */
  int64_t n_global;
  int64_t row_begin, row_end;
  const int32_t* row_ptr;  /* CSR only */
  const int32_t* col_idx;  /* CSR only */
  const double* val;       /* CSR only */
  int64_t nnz_local;       /* CSR only: row_ptr[last] */
} sks_operator;

/* ---- sketched GMRES (Alg. 1 + iterative sGMRES + restarting) ------------------ */

typedef struct {
  int32_t d;        /* basis columns per cycle */
  int32_t k;        /* partial-orthogonalisation window, 1 <= k <= 8 */
  int32_t s;        /* sketch rows, d+1 <= s <= 2048 */
  int32_t zeta;     /* nonzeros per column of S, 1 <= zeta <= min(s, 16) */
  uint64_t seed;    /* S hash seed (S differs per cycle, reading O7) */
  double tol;       /* stop when ||f - A x||_2 / ||f||_2 <= tol (true residual, O16) */
  int32_t max_cycles;        /* restarts (O17) */
  int32_t sketch_batch;      /* columns per sketch batch, 0 = default (32), <= 32 */
  double early_exit_factor;  /* in-cycle exit when r_est,j <= factor*tol*||f|| (O16); 0 = never */
  double cond_tol;           /* kappa(T) warning threshold, default 1e14 */
  int32_t flags;             /* SKS_OPT_* bits */
  int32_t time_stride;       /* SKS_OPT_TIME_STEPS: time every time_stride-th step launch (0/1 = all); for
                                stencil operators with time_stride > 1 one event pair brackets a window of
                                time_stride consecutive launches inside a sketch batch (SKS_TIME_WINDOW=n:
                                windows of n, 1 = single launches) */
  int32_t basis;             /* SKS_BASIS_ARNOLDI (k-truncated, Eq. partorth) or SKS_BASIS_CHEBYSHEV */
  int32_t sketch;            /* SKS_SKETCH_SPARSE (Eq. sparse-map) or SKS_SKETCH_SRFT (Eq. SRFT, single GPU) */
  double cheb_c, cheb_dx, cheb_dy;  /* Chebyshev: spectrum inside [c +- dx] x [+- i dy];
                                       all 0 = closed-form box of the stencil operator */
} sks_sgmres_opts;

enum {
  SKS_SKETCH_SPARSE = 0,  /* sparse sign map, Eq. (sparse-map), hashed (readings O1-O7) */
  SKS_SKETCH_SRFT = 1     /* SRFT, Eq. (SRFT) P:631-638 with F = orthonormal DCT2 as in the paper's
                             experiments: S x = sqrt(n/s) DCT2(E x)[q_0..q_{s-1}], hashed signs E
                             and Floyd-sampled coordinates q (reading O32).  The DCT mixes all rows: nranks = 1
                             only (SKS_EUNSUPPORTED otherwise).  zeta is ignored. */
};

enum {
  SKS_BASIS_ARNOLDI = 0,   /* k-partial Arnoldi, Eq. (partorth) */
  SKS_BASIS_CHEBYSHEV = 1, /* shifted-scaled Chebyshev recurrence, Eq. (Chebrecurse) P:1192-1199,
                              vectors rescaled to unit norm after use; no inner
                              products in the recurrence (stencil operators only) */
  SKS_BASIS_BLOCK_CHEBYSHEV = 2 /* sks_srr_eigs only: block Chebyshev basis of the block Krylov space
                              K_p(A; Omega), Sec. "Block Krylov subspaces" P:1867-1896 and "Block Chebyshev
                              recurrence" P:1983-2008: B_1 = Omega (v0 holds the n_local x b start block,
                              column-major), B_2 = (A - cI) B_1 / (2 rho), B_j = [(A - cI) B_{j-1}
                              - (dx^2 - dy^2)/(4 rho) B_{j-2}] / rho; block size b = opts.block, depth
                              p = d / b (d must be a multiple of b); no normalisation, no inner products;
                              S A B from the sketched B_{p+1} through the recurrence (reading O34); stencil
                              operators only (SKS_EUNSUPPORTED for CSR) */
};

enum {
  SKS_OPT_TIME_STEPS = 1,       /* bracket every basis-step launch with CUDA events on the main stream and
                                   report the summed kernel time in info->t_step_s (measurement only) */
  SKS_OPT_ZERO_X0 = 4,          /* x0 = 0: x is output only (its input content is not read or copied) */
  SKS_OPT_WHITEN = 8,           /* whitening instead of restarting (Fact "Whitening" P:598-612; P:1398-1400
                                   "approximately orthogonalize B by replacing it with B T^{-1}"; reading O36):
                                   when first kappa_2(T_j) > cond_tol, the first J = j-1 columns become
                                   B_J T_J^{-1} (unit columns), T_J its diagonal, and the basis continues from
                                   them; a second crossing at the same J ends the cycle.  k-truncated Arnoldi on
                                   stencil operators (SKS_EUNSUPPORTED otherwise); info->flags SKS_INFO_WHITEN */
  SKS_OPT_ADAPTIVE_RESTART = 2  /* adaptive restarting (Sec. "Adaptive restarting"): when
                                   first kappa_2(T_j) > cond_tol, the cycle ends with the previous
                                   solution (j-1 columns) and restarts from its residual (reading O31:
                                   kappa_2 estimated by power iteration on the device, checked after
                                   every sketched-QR batch, the first j located by bisection) */
};

typedef struct {
  int32_t cycles;       /* cycles run */
  int32_t columns;      /* basis columns used in solutions (sum over cycles) */
  int32_t columns_generated; /* basis columns generated (>= columns: batches run ahead) */
  int32_t flags;        /* SKS_WARN_* */
  double rel_res_true;  /* ||f - A x|| / ||f|| at exit (recomputed on device) */
  double r_est;         /* last sketched residual estimate / ||f|| */
  double cond_T;        /* kappa_2(T) of the last cycle's triangular factor (power-iteration estimate) */
  double t_total_s;     /* device time of the whole call (events on the main stream) */
  double t_basis_s;     /* device time of the basis loops (step kernels, all cycles) */
  double bytes_basis;   /* algorithmic HBM bytes of the basis loops */
  int64_t kernel_launches; /* CUDA kernels this call launched */
  int64_t steps;        /* step-kernel launches (one per basis column) */
  double t_step_s;      /* SKS_OPT_TIME_STEPS: summed duration of the step launches (events), else 0 */
  int64_t steps_timed;  /* step launches included in t_step_s */
  double bytes_step;    /* algorithmic HBM bytes of those launches */
} sks_sgmres_info;

/* Solve A x = f.  f, x: this rank's rows (n_local = row_end - row_begin); x is in/out
 * (x0 in, solution out).  hist: caller buffer of hist_cap doubles receiving
 * r_est,j/||f|| for every used column of every cycle, concatenated (may be NULL);
 * hist_true: hist_true_cap doubles receiving ||f-Ax||/||f|| after each cycle (may
 * be NULL).  Returns SKS_OK when the tolerance was met, SKS_ENOTCONV otherwise. */
sks_status sks_sgmres_solve(sks_ctx* ctx, const sks_operator* A, const double* f, double* x,
                            const sks_sgmres_opts* opts, sks_sgmres_info* info,
                            double* hist, int64_t hist_cap,
                            double* hist_true, int64_t hist_true_cap);

/* ---- sketched Rayleigh-Ritz (Alg. 2) ------------------------------------------ */

typedef struct {
  int32_t d, k, s, zeta;
  uint64_t seed;
  double cond_tol;
  int32_t basis;        /* SKS_BASIS_* */
  int32_t sketch;       /* SKS_SKETCH_* */
  int32_t stabilize;    /* SKS_SRR_STABILIZE_* (Sec. "Stabilization"; reading O33) */
  int32_t block;        /* SKS_BASIS_BLOCK_CHEBYSHEV: block size b >= 1 (d = b p); ignored otherwise */
  double cheb_c, cheb_dx, cheb_dy;  /* as in sks_sgmres_opts */
} sks_srr_opts;

/* Stabilised sRR (Alg. 2 P:1679-1681 "stabilize and solve (eq:qz)"): truncated SVD
 * SB = U Sigma V^* + E keeping sigma_i >= sigma_1 / cond_tol (rank r, reported in info->rank), then
 * the r x r pencil (U^* SAB V) z = theta Sigma z; y = V z, x = B y.  Computed by a one-sided
 * Jacobi SVD of SB in one CTA, M_r = Sigma_r^-1 U_r^T SAB V_r and the Francis QR of M_r (Sigma_r
 * is diagonal with kappa <= cond_tol, reading O33).
 * OFF: never; IF_ILL: when the kappa_2(T) estimate exceeds cond_tol (Alg. 2's test); ALWAYS. */
enum { SKS_SRR_STABILIZE_OFF = 0, SKS_SRR_STABILIZE_IF_ILL = 1, SKS_SRR_STABILIZE_ALWAYS = 2 };

typedef struct {
  int32_t columns;
  int32_t flags;
  int32_t nev_out;      /* pairs written: nev, or nev+1 when position nev splits a conjugate pair (O23) */
  int32_t rank;         /* columns of the Rayleigh-Ritz problem: de (unstabilised) or the truncated rank r */
  double cond_SB;       /* kappa_2 estimate of the triangular factor of SB */
  double t_total_s, t_basis_s, t_small_s;
  double bytes_basis;
  int64_t kernel_launches;
  int64_t steps;
} sks_srr_info;

/* v0: start vector rows of this rank.  Outputs (caller-owned, capacity nev_cap >=
 * nev+1): theta_re/theta_im (order: |theta| descending, ties Im descending, O23),
 * res_true = ||A x - theta x||/||x|| with x = B y (O24), res_est (Eq. srr-resid-est).
 * X_re/X_im: n_local x nev_cap column-major Ritz vectors (may be NULL). */
sks_status sks_srr_eigs(sks_ctx* ctx, const sks_operator* A, const double* v0,
                        const sks_srr_opts* opts, int32_t nev, int32_t nev_cap,
                        double* theta_re, double* theta_im, double* res_true, double* res_est,
                        double* X_re, double* X_im, sks_srr_info* info);

/* ---- test / parity entry points ------------------------------------------------ */

/* SM = S_cycle M for this rank's rows (global rows [row_begin,row_end)), reduced over
 * ranks.  M: n_local x c column-major with leading dimension ldm; SM: s x c
 * column-major (ld = s).  S per the hash spec of SPEC "S hash" in DESIGN.md. */
sks_status sks_sketch_apply(sks_ctx* ctx, int64_t n_global, int64_t row_begin, int64_t row_end,
                            int32_t s, int32_t zeta, uint64_t seed, uint32_t cycle,
                            const double* M, int64_t ldm, int32_t c, double* SM);

/* S M for the SRFT sketch (SKS_SKETCH_SRFT, reading O32) of cycle `cycle`: M is n x c column-major
 * (host or device), SM is s x c column-major (host or device, caller-owned).  Single rank only.
 * Errors: SKS_EINVAL (n < 1, s < 1, s > n, c < 1, NULL), SKS_EUNSUPPORTED (nranks > 1). */
sks_status sks_srft_apply(sks_ctx* ctx, int64_t n, int32_t s, uint64_t seed, uint32_t cycle, const double* M,
                          int32_t c, double* SM);

/* (row, sign) table of S for global rows [row_begin, row_begin+count), computed ON
 * THE DEVICE by the same code the sketch kernel uses: q[count*zeta] int32 in [0,s),
 * sign[count*zeta] int8 (+1/-1), row-major (row, t). */
sks_status sks_sketch_table(sks_ctx* ctx, int64_t row_begin, int64_t count, int32_t s,
                            int32_t zeta, uint64_t seed, uint32_t cycle,
                            int32_t* q, int8_t* sign);

/* y = A x on this rank's rows (halo exchanged internally). */
sks_status sks_apply_operator(sks_ctx* ctx, const sks_operator* A, const double* x, double* y);

/* First ncols columns of the k-truncated Arnoldi basis started from r0
 * (b_0 = r0/||r0||), normalised, n_local x ncols column-major (ld = n_local),
 * and Hbar ((ncols) x (ncols-1) column-major, ld = ncols): the recurrence
 * A B[:, :ncols-1] = B Hbar, entries h_{ij} = <b_i, A b_j> (i in window) and
 * Hbar[j+1, j] = ||w_{j+1}||.  H_out may be NULL. */
sks_status sks_basis(sks_ctx* ctx, const sks_operator* A, const double* r0, int32_t k,
                     int32_t ncols, double* B_out, double* H_out);

#ifdef __cplusplus
}
#endif

#endif /* SKS_H */
