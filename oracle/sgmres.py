"""sGMRES -- oracle side.  Alg. 1, iterative sGMRES,
restarting.

One cycle c (Alg. 1 + P:1351-1385, readings O7, O13, O14, O16):
  1. r = f - A x;  g = S_c r
  2. b_1 = r/||r||, m_1 = A b_1; k-partial Arnoldi to d
  3. C = S_c [m_1 ... m_d]                                 ("Sketch reduced matrix")
  4. thin QR  C = U T, T diagonal >= 0                     (Eq. sgmres-yhat)
  5. r_est,j = ||(I - U_j U_j^T) g||, j = 1..d             (Eq. sgmres-iterative-soln, O14)
     first j with r_est,j <= early_exit_factor * tol * ||f|| (O16), else j = d
  6. yhat_j = T_j^{-1} (U_j^T g)                           (Eq. sgmres-iterative-soln)
  7. x <- x + B_j yhat_j                                   (O13: x0 + B yhat, not "+ [m_1..m_j] yhat")
  kappa_2(T_j) recorded; > cond_tol sets the warning flag.
Cycles repeat with a fresh S_{c+1} while ||f - A x||/||f|| > tol, up to max_cycles
(O15, O17).  Convergence is judged on the TRUE residual (O16).
"""
import numpy as np
from scipy.linalg import solve_triangular

from .krylov import partial_arnoldi, chebyshev_basis
from .sketch import sketch_matrix, SRFT

WARN_COND = 1
WARN_BREAKDOWN = 2
INFO_ADAPTIVE = 8   # adaptive restarting ended a cycle early


def thin_qr(C):
    """Thin QR C = U T with T upper triangular, diag(T) >= 0."""
    Q, R = np.linalg.qr(C, mode="reduced")
    sgn = np.sign(np.diag(R))
    sgn[sgn == 0] = 1.0
    return Q * sgn[None, :], R * sgn[:, None]


def gmres_exact_ls(M, r0):
    """GMRES problem over the same basis: min ||AB y - r0|| (Eq. gmres)."""
    y, *_ = np.linalg.lstsq(M, r0, rcond=None)
    return y


def sgmres_cycle(matvec, f, x, d, k, s, zeta, seed, cycle, tol=1e-8,
                 early_exit_factor=0.25, cond_tol=1e14, fnorm=None, S=None, cheb=None, adaptive=False,
                 sketch="sparse"):
    """One cycle; cheb = (c, dx, dy) selects the Chebyshev basis of Eq. Chebrecurse
     instead of k-truncated Arnoldi.
    adaptive: adaptive restarting (Sec. adaptive-restart): "When first
    kappa_2(T_j) > tol, we recognize that it is time to restart.  We generate the new Krylov
    subspace using the previous residual r_{j-1} = r_0 - AB_{j-1} y_{j-1}" -- the cycle keeps
    the solution of j-1 columns (at least one column is always used)."""
    f = np.asarray(f, dtype=np.float64)
    n = f.size
    if fnorm is None:
        fnorm = np.linalg.norm(f)
    if S is None:  # sketch: "sparse" (Eq. sparse-map) or "srft" (Eq. SRFT with DCT2, reading O32)
        S = sketch_matrix(n, s, zeta, seed, cycle) if sketch == "sparse" else SRFT(n, s, seed, cycle)
    r = f - matvec(x)
    if np.linalg.norm(r) == 0.0:
        return dict(x=x.copy(), j=0, r_est=np.zeros(0), yhat=np.zeros(0),
                    cond_T=1.0, flags=0, basis=None, C=None, g=None)
    g = S @ r
    basis = partial_arnoldi(matvec, r, d, k) if cheb is None else chebyshev_basis(matvec, r, d, *cheb)
    B, M, de = basis["B"], basis["M"], basis["d_eff"]
    C = S @ M
    U, T = thin_qr(C)
    c = U.T @ g
    r_est = np.empty(de)
    for j in range(1, de + 1):
        r_est[j - 1] = np.linalg.norm(g - U[:, :j] @ c[:j])
    thr = early_exit_factor * tol * fnorm
    hits = np.nonzero(r_est <= thr)[0] if early_exit_factor > 0 else np.zeros(0, int)
    jstar = int(hits[0]) + 1 if hits.size else de
    adapted = False
    if adaptive:
        conds = np.array([np.linalg.cond(T[:j, :j]) for j in range(1, de + 1)])   # exact 2-norm
        over = np.nonzero(conds > cond_tol)[0]
        if over.size:
            jfirst = int(over[0]) + 1
            if max(jfirst - 1, 1) < jstar:
                jstar = max(jfirst - 1, 1)
                adapted = True
    yhat = solve_triangular(T[:jstar, :jstar], c[:jstar], lower=False)
    x_new = x + B[:, :jstar] @ yhat
    condT = np.linalg.cond(T[:jstar, :jstar])
    flags = (WARN_COND if condT > cond_tol else 0) | (WARN_BREAKDOWN if basis["breakdown"] else 0) | \
        (INFO_ADAPTIVE if adapted else 0)
    return dict(x=x_new, j=jstar, r_est=r_est[:jstar], yhat=yhat, cond_T=condT,
                flags=flags, basis=basis, C=C, g=g, U=U, T=T)


def sgmres_solve(matvec, f, d, k, s, zeta, seed, tol=1e-8, max_cycles=50,
                 early_exit_factor=0.25, cond_tol=1e14, x0=None, keep_last=False, cheb=None, adaptive=False,
                 sketch="sparse"):
    """Restarted sGMRES.  Returns dict(x, cycles, columns, rel_res_true, r_est,
    hist_est (r_est_j/||f|| per column, concatenated), hist_true (per cycle),
    cond_T, flags)."""
    f = np.asarray(f, dtype=np.float64)
    fnorm = np.linalg.norm(f)
    x = np.zeros_like(f) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    hist_est, hist_true = [], []
    columns, flags, condT, r_est = 0, 0, 1.0, np.nan
    last = None
    cycles = 0
    for c in range(max_cycles):
        out = sgmres_cycle(matvec, f, x, d, k, s, zeta, seed, c, tol,
                           early_exit_factor, cond_tol, fnorm, cheb=cheb, adaptive=adaptive, sketch=sketch)
        cycles += 1
        x = out["x"]
        columns += out["j"]
        flags |= out["flags"]
        condT = out["cond_T"]
        if out["j"]:
            r_est = out["r_est"][-1]
        hist_est.extend((out["r_est"] / fnorm).tolist())
        rel = np.linalg.norm(f - matvec(x)) / fnorm
        hist_true.append(rel)
        last = out
        if rel <= tol:
            break
    res = dict(x=x, cycles=cycles, columns=columns, rel_res_true=hist_true[-1],
               r_est=r_est, hist_est=np.array(hist_est), hist_true=np.array(hist_true),
               cond_T=condT, flags=flags)
    if keep_last:
        res["last"] = last
    return res
