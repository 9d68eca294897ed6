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
INFO_WHITEN = 32    # the basis was whitened at least once (Fact "Whitening" P:598-612)


def thin_qr(C):
    """Thin QR C = U T with T upper triangular, diag(T) >= 0."""
    Q, R = np.linalg.qr(C, mode="reduced")
    sgn = np.sign(np.diag(R))
    sgn[sgn == 0] = 1.0
    return Q * sgn[None, :], R * sgn[:, None]


def whitened_basis(matvec, r, d, k, S, cond_tol, breakdown_tol=1e-14, record=False):
    """k-truncated Arnoldi (Eq. partorth) with WHITENING instead of restarting (P:1398-1400:
    "instead of restarting, we could approximately orthogonalize B by replacing it with B T^{-1}, whose
    condition number is constant"; Fact "Whitening" P:598-612), reading O36:
      after each new column b_j, thin QR  S [A b_0 ... A b_j] = U T;  when first kappa_2(T) > cond_tol, the
      columns b_0..b_{j-1} (those before the new one, J = j of them) are replaced by B_J T_J^{-1} (and A B_J by
      A B_J T_J^{-1}, the same linear map), the new column is discarded, and the recurrence continues from the
      whitened columns (b_J regenerated from A b_{J-1} against the last k whitened columns).  If the threshold is
      crossed again at the same J (no progress since the last whitening), generation stops with J columns.
    The whitened columns are rescaled to unit 2-norm, like every basis vector (the sketched QR's
    kappa_2(T) is not invariant to column scaling, and a unit new column next to whitened columns of norm
    ~ 1/||A|| would cross the threshold through scaling alone).  T_J^{-1} is applied with a triangular solve.  Returns dict(B, M = A B, d_eff, events (the J of each
    whitening), breakdown, stopped, snapshots: [(J, A B_J T_J^{-1})] when record)."""
    r = np.asarray(r, dtype=np.float64)
    rho = np.linalg.norm(r)
    B = [r / rho]
    M = [matvec(B[0])]
    events, snaps = [], []
    last, breakdown, stopped = -1, False, False
    while len(B) < d:
        j = len(B)
        lo = max(0, j - k)
        W = np.stack(B[lo:j], axis=1)
        m = M[j - 1]
        h = W.T @ m                        # classical Gram-Schmidt from the same m (reading O8)
        w = m - W @ h
        nu = np.linalg.norm(w)
        if nu <= breakdown_tol * np.linalg.norm(m):
            breakdown = True
            break
        B.append(w / nu)
        M.append(matvec(B[-1]))
        _, T = thin_qr(S @ np.stack(M, axis=1))
        if np.linalg.cond(T) > cond_tol:
            B.pop()
            M.pop()
            if j <= last:
                stopped = True
                break
            Tinv = solve_triangular(T[:j, :j], np.eye(j), lower=False)
            Bw = np.stack(B, axis=1) @ Tinv
            Mw = np.stack(M, axis=1) @ Tinv
            if record:
                snaps.append((j, Mw.copy()))   # A B_J T_J^{-1}, before the rescaling
            nrm = np.linalg.norm(Bw, axis=0)   # unit columns, as every basis vector
            Bw /= nrm[None, :]
            Mw /= nrm[None, :]
            B = [Bw[:, i] for i in range(j)]
            M = [Mw[:, i] for i in range(j)]
            events.append(j)
            last = j
    return dict(B=np.stack(B, axis=1), M=np.stack(M, axis=1), d_eff=len(B), events=events, breakdown=breakdown,
                stopped=stopped, snapshots=snaps)


def gmres_exact_ls(M, r0):
    """GMRES problem over the same basis: min ||AB y - r0|| (Eq. gmres)."""
    y, *_ = np.linalg.lstsq(M, r0, rcond=None)
    return y


def sgmres_cycle(matvec, f, x, d, k, s, zeta, seed, cycle, tol=1e-8,
                 early_exit_factor=0.25, cond_tol=1e14, fnorm=None, S=None, cheb=None, adaptive=False,
                 sketch="sparse", whiten=False):
    """One cycle; cheb = (c, dx, dy) selects the Chebyshev basis of Eq. Chebrecurse
     instead of k-truncated Arnoldi.
    adaptive: adaptive restarting (Sec. adaptive-restart): "When first
    kappa_2(T_j) > tol, we recognize that it is time to restart.  We generate the new Krylov
    subspace using the previous residual r_{j-1} = r_0 - AB_{j-1} y_{j-1}" -- the cycle keeps
    the solution of j-1 columns (at least one column is always used).
    whiten: whitening instead of restarting (whitened_basis, reading O36)."""
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
    if whiten:
        basis = whitened_basis(matvec, r, d, k, S, cond_tol)
    else:
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
        (INFO_ADAPTIVE if adapted else 0) | (INFO_WHITEN if basis.get("events") else 0)
    return dict(x=x_new, j=jstar, r_est=r_est[:jstar], yhat=yhat, cond_T=condT,
                flags=flags, basis=basis, C=C, g=g, U=U, T=T)


def sgmres_solve(matvec, f, d, k, s, zeta, seed, tol=1e-8, max_cycles=50,
                 early_exit_factor=0.25, cond_tol=1e14, x0=None, keep_last=False, cheb=None, adaptive=False,
                 sketch="sparse", whiten=False):
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
                           early_exit_factor, cond_tol, fnorm, cheb=cheb, adaptive=adaptive, sketch=sketch,
                           whiten=whiten)
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
