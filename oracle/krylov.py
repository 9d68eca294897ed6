"""Krylov bases -- oracle side.

partial_arnoldi: Arnoldi with k-partial orthogonalisation, Eq. (partorth)
P:208-218 and Alg. 1 lines P:1296-1307:
    b_1 = r/||r||, m_1 = A b_1;  for j = 2..d:
    w_j = (I - b_{j-1}b_{j-1}^* - ... - b_{j-k}b_{j-k}^*) m_{j-1}   (b_{-i} = 0)
    b_j = w_j/||w_j||,  m_j = A b_j.
Reading O8: the sum form with all coefficients h_i = <b_i, m_{j-1}> taken from the
same m_{j-1} (classical Gram-Schmidt, one pass), exactly as the display reads.
Reading O10: breakdown when ||w_j|| <= 1e-14 ||m_{j-1}||; the basis stops at j-1.
H records the recurrence: A B[:, :j] = B[:, :j+1] Hbar, i.e.
  m_{j-1} = sum_i h_i b_i + ||w_j|| b_j  ->  Hbar[i, j-1] = h_i, Hbar[j, j-1] = ||w_j||
(0-based column j-1 of Hbar belongs to m_{j-1}).

full_arnoldi: the classic process of P:1081-1099 (q_{j+1} from (I - Q_j Q_j^*) A q_j),
with two Gram-Schmidt passes ("Robust implementations usually incorporate double
Gram-Schmidt").  Used only as a baseline in pins.
"""
import numpy as np


def partial_arnoldi(matvec, r, d: int, k: int, breakdown_tol: float = 1e-14):
    """Return dict(B (n x d_eff), M = AB (n x d_eff), H ((d_eff+1) x d_eff with the
    last row filled only if the next column was formed), d_eff, breakdown, nu)."""
    r = np.asarray(r, dtype=np.float64)
    n = r.size
    B = np.zeros((n, d))
    M = np.zeros((n, d))
    H = np.zeros((d + 1, d))
    rho = np.linalg.norm(r)
    B[:, 0] = r / rho
    M[:, 0] = matvec(B[:, 0])
    d_eff = d
    breakdown = False
    for j in range(1, d):                  # 0-based j is the paper's j+1
        lo = max(0, j - k)
        W = B[:, lo:j]
        m = M[:, j - 1]
        h = W.T @ m                        # all h from the same m_{j-1}
        w = m - W @ h
        nu = np.linalg.norm(w)
        H[lo:j, j - 1] = h
        H[j, j - 1] = nu
        if nu <= breakdown_tol * np.linalg.norm(m):
            d_eff = j
            breakdown = True
            break
        B[:, j] = w / nu
        M[:, j] = matvec(B[:, j])
    return dict(B=B[:, :d_eff], M=M[:, :d_eff], H=H[:d_eff + 1, :d_eff],
                d_eff=d_eff, breakdown=breakdown, rho=rho)


def partial_arnoldi_next(matvec, B, M, k: int):
    """One more column b_{d+1} (and its h, nu) after a partial_arnoldi basis: the
    column of Hbar belonging to m_d.  Returns (b_next, h (len d), nu)."""
    d = B.shape[1]
    lo = max(0, d - k)
    m = M[:, d - 1]
    W = B[:, lo:d]
    h_w = W.T @ m
    w = m - W @ h_w
    nu = np.linalg.norm(w)
    h = np.zeros(d)
    h[lo:d] = h_w
    return w / nu, h, nu


def full_arnoldi(matvec, r, p: int):
    r = np.asarray(r, dtype=np.float64)
    n = r.size
    Q = np.zeros((n, p + 1))
    H = np.zeros((p + 1, p))
    Q[:, 0] = r / np.linalg.norm(r)
    for j in range(p):
        w = matvec(Q[:, j])
        for _ in range(2):
            c = Q[:, :j + 1].T @ w
            w = w - Q[:, :j + 1] @ c
            H[:j + 1, j] += c
        H[j + 1, j] = np.linalg.norm(w)
        if H[j + 1, j] == 0.0:
            return Q[:, :j + 1], H[:j + 2, :j + 1]
        Q[:, j + 1] = w / H[j + 1, j]
    return Q, H


def chebyshev_basis(matvec, r, d: int, c: float, dx: float, dy: float = 0.0):
    """Shifted-and-scaled Chebyshev basis, Eq. (Chebrecurse) P:1192-1199:
        b_1 = r/||r||,  b_2 = (2 rho)^-1 (A - c I) b_1,
        b_j = rho^-1 [ (A - c I) b_{j-1} - (dx^2 - dy^2)/(4 rho) b_{j-2} ],  j = 3..d,
    rho = max(dx, dy), for a spectrum inside the rectangle [c +- dx, +- i dy].  "In practice, we
    also rescale each basis vector b_j to have unit norm after it has played its role in the
    recurrence": the recurrence runs on the raw vectors, the returned basis holds
    them normalised.  No inner products.
    Returns dict(B (n x d, unit columns), M = A B, raw (n x d raw recurrence vectors),
    H ((d+1) x d): A B[:, :d-1] = B H[:d, :d-1] (recurrence identity), d_eff, rho, rnorm)."""
    r = np.asarray(r, dtype=np.float64)
    n = r.size
    rho = max(dx, dy)
    e = (dx * dx - dy * dy) / (4.0 * rho)
    raw = np.zeros((n, d))
    rnorm = np.linalg.norm(r)
    raw[:, 0] = r / rnorm
    Ab = [matvec(raw[:, 0])]
    if d >= 2:
        raw[:, 1] = (Ab[0] - c * raw[:, 0]) / (2.0 * rho)
    for j in range(2, d):
        Ab.append(matvec(raw[:, j - 1]))
        raw[:, j] = (Ab[j - 1] - c * raw[:, j - 1] - e * raw[:, j - 2]) / rho
    if d >= 2:
        Ab.append(matvec(raw[:, d - 1]))
    nu = np.linalg.norm(raw, axis=0)
    B = raw / nu[None, :]
    M = np.stack([a / nu[j] for j, a in enumerate(Ab[:d])], axis=1)
    # recurrence identity on the normalised basis: A raw_0 = 2 rho raw_1 + c raw_0,
    # A raw_j = rho raw_{j+1} + c raw_j + e raw_{j-1}  (j >= 1)
    H = np.zeros((d + 1, d))
    for j in range(d - 1):
        lead = 2.0 * rho if j == 0 else rho
        H[j + 1, j] = lead * nu[j + 1] / nu[j]
        H[j, j] = c
        if j >= 1:
            H[j - 1, j] = e * nu[j - 1] / nu[j]
    return dict(B=B, M=M, raw=raw, H=H, d_eff=d, rho=rho, rnorm=rnorm, breakdown=False, nu=nu)


def block_chebyshev_basis(matvec, Omega, p: int, c: float, dx: float, dy: float = 0.0):
    """Block Chebyshev basis for the block Krylov space K_p(A; Omega), Sec. "Block Chebyshev recurrence"
    (P:1983-2008), written out exactly as displayed:
        B_1 = Omega;   B_2 = (2 rho)^-1 (A - c I) Omega;
        B_j = rho^-1 [ (A - c I) B_{j-1} - (dx^2 - dy^2)/(4 rho) B_{j-2} ],   j = 3..p,
    rho = max(dx, dy), for a spectrum inside [c +- dx, +- i dy].  No inner products, no orthogonalisation and
    no rescaling (the paper's display has none; sRR is invariant to column scaling of B).
    Omega: n x b.  Returns dict(B (n x bp; block j in columns [(j-1) b, j b)), M = A B computed column by
    column with the operator (the plain definition of AB), b, p, rho)."""
    Omega = np.asarray(Omega, dtype=np.float64)
    if Omega.ndim == 1:
        Omega = Omega[:, None]
    n, b = Omega.shape
    rho = max(dx, dy)
    e = (dx * dx - dy * dy) / (4.0 * rho)

    def apply(X):
        return np.stack([matvec(X[:, i]) for i in range(X.shape[1])], axis=1)

    blocks = [Omega.copy()]
    if p >= 2:
        blocks.append((apply(blocks[0]) - c * blocks[0]) / (2.0 * rho))
    for j in range(2, p):
        blocks.append((apply(blocks[j - 1]) - c * blocks[j - 1] - e * blocks[j - 2]) / rho)
    B = np.concatenate(blocks, axis=1)
    M = apply(B)
    return dict(B=B, M=M, b=b, p=p, rho=rho, e=e)
