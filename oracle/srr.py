"""Sketched Rayleigh-Ritz -- oracle side.  Alg. 2, Eq. Mhat-form
(P:1598-1601), Eq. srr-resid-est.

  b_1 = v0/||v0||; k-partial Arnoldi to d columns
  C = S B,  D = S AB   (one shared S)                      (O11)
  thin QR  C = U T
  Mhat = T^{-1} (U^T D)                                    (Eq. Mhat-form; O22)
  eig(Mhat) -> (theta_i, y_i)                              ("the QR algorithm" P:1603)
  r_est,i = ||D y_i - theta_i C y_i|| / ||C y_i||          (Eq. srr-resid-est)
  x_i = B y_i;  true residual ||A x_i - theta_i x_i|| / ||x_i||   (O24; no tau filter)
Selection (O23): nev pairs of largest |theta|, ties broken by Im(theta)
descending; if position nev splits a conjugate pair, the partner is included.

Stabilised sRR (Sec. "Stabilization"; Alg. 2; reading O33):
  truncated SVD  C = U Sigma V^* + E, keeping sigma_i >= sigma_1 / tol
  QZ on the pencil (U^* D V) z = theta Sigma z                          (Eq. qz)
  y = V z, x = B y  (the "sRR eigenpair (Vz, theta)")
stabilize = "off" | "if_ill" (kappa_2(T) > tol, Alg. 2's test) | "always".
"""
import numpy as np
from scipy.linalg import eig as qz_eig, solve_triangular

from .krylov import partial_arnoldi, block_chebyshev_basis
from .sgmres import thin_qr
from .sketch import sketch_matrix, SRFT


def select_ritz(theta, nev):
    """Indices of the nev largest-|theta| Ritz values, canonical order (O23)."""
    theta = np.asarray(theta)
    # lexsort: last key primary -> sort by -|theta| then by -Im
    order = np.lexsort((-theta.imag, -np.abs(theta)))
    sel = list(order[:nev])
    if nev < len(order):
        last = theta[order[nev - 1]]
        nxt = theta[order[nev]]
        if last.imag != 0.0 and np.isclose(nxt, np.conj(last), rtol=1e-12, atol=0.0):
            sel.append(order[nev])
    return np.array(sel, dtype=np.int64)


def stabilized_pencil(C, D, tol):
    """Truncated SVD of C = SB and the generalized eigenproblem (U^* D V) z = theta Sigma z solved by
    QZ (scipy's ggev).  Returns theta (all r), Y = V Z and the rank r."""
    Uc, sig, Vh = np.linalg.svd(C, full_matrices=False)
    r = int(np.count_nonzero((sig > 0) & (sig * tol >= sig[0])))
    Ur, Vr = Uc[:, :r], Vh[:r].T
    theta, Z = qz_eig(Ur.T @ D @ Vr, np.diag(sig[:r]))
    return theta, Vr @ Z, r, sig


def srr_from_basis(matvec, B, M, S, nev, stabilize="off", tol=1e14):
    C = S @ B
    D = S @ M
    U, T = thin_qr(C)
    cond_T = np.linalg.cond(T)
    stab = stabilize == "always" or (stabilize == "if_ill" and cond_T > tol)
    rank, sig = C.shape[1], None
    if stab:
        Mhat = None
        theta, Y, rank, sig = stabilized_pencil(C, D, tol)
    else:
        Mhat = solve_triangular(T, U.T @ D, lower=False)
        theta, Y = np.linalg.eig(Mhat)
    sel = select_ritz(theta, min(nev, len(theta)))
    th = theta[sel]
    Ys = Y[:, sel]
    res_est = np.array([np.linalg.norm(D @ y - t * (C @ y)) / np.linalg.norm(C @ y)
                        for t, y in zip(th, Ys.T)])
    X = B @ Ys
    res_true = np.empty(len(sel))
    for i in range(len(sel)):
        x = X[:, i]
        Ax = matvec(x.real) + 1j * matvec(x.imag)
        res_true[i] = np.linalg.norm(Ax - th[i] * x) / np.linalg.norm(x)
    return dict(theta=th, Y=Ys, X=X, res_est=res_est, res_true=res_true,
                Mhat=Mhat, C=C, D=D, U=U, T=T, cond_SB=np.linalg.cond(C),
                theta_all=theta, stabilized=stab, rank=rank, sigma=sig)


def srr_eigs(matvec, v0, d, k, s, zeta, seed, nev, cycle=0, sketch="sparse", stabilize="off", tol=1e14):
    """sketch: "sparse" (Eq. sparse-map, O1-O7) or "srft" (Eq. SRFT with DCT2, O32);
    stabilize/tol: stabilised sRR (O33)."""
    v0 = np.asarray(v0, dtype=np.float64)
    n = v0.size
    basis = partial_arnoldi(matvec, v0, d, k)
    S = sketch_matrix(n, s, zeta, seed, cycle) if sketch == "sparse" else SRFT(n, s, seed, cycle)
    out = srr_from_basis(matvec, basis["B"], basis["M"], S, nev, stabilize, tol)
    out["basis"] = basis
    return out


def srr_eigs_block(matvec, Omega, p, c, dx, dy, s, zeta, seed, nev, cycle=0, stabilize="off", tol=1e14):
    """sRR with the block Chebyshev basis of Sec. "Block Krylov subspaces" / "Block Chebyshev recurrence"
    (P:1867-1896): B = [B_1 ... B_p] from the start block Omega (n x b, "drawn at random from a
    standard normal distribution"), then Alg. 2's sketch, QR, Mhat, eigenpairs and residuals
    (srr_from_basis, one shared S) exactly as for the single-vector basis (d = b p)."""
    bas = block_chebyshev_basis(matvec, Omega, p, c, dx, dy)
    n = bas["B"].shape[0]
    S = sketch_matrix(n, s, zeta, seed, cycle)
    out = srr_from_basis(matvec, bas["B"], bas["M"], S, nev, stabilize, tol)
    out["basis"] = bas
    return out
