"""Operators A of the BASELINE.json configs, written from their definitions.

Convection-diffusion  -Laplace(u) + beta (d/dx + d/dy [+ d/dz]) u  on the unit
square/cube, m interior points per side, h = 1/(m+1), homogeneous Dirichlet,
centred differences (BASELINE.json configs; reading SURVEY 8(c) O18).
Row order r = i + m*j (+ m^2*l), x fastest, 0-based.

The oracle builds A as a Kronecker sum of the 1D tridiagonal factor
    T = tridiag(b, a, c),  a = 2/h^2,  b = -1/h^2 - beta/(2h),  c = -1/h^2 + beta/(2h)
    A_2D = I (x) T + T (x) I,   A_3D = I(x)I(x)T + I(x)T(x)I + T(x)I(x)I
which is the same matrix as the 5-/7-point stencil (pinned in tests against an
explicit loop over grid points), and is independent of the GPU's matrix-free
stencil.  The unscaled form (multiplied through by nothing) is used, i.e. the
entries carry the 1/h^2 and 1/(2h) factors exactly as in O18.

Closed form (BASELINE north_star, "a+2 sqrt(bc) cos(j pi/(n+1))"): eigenvalues of T
are  mu_p = a + 2 sqrt(b c) cos(p pi/(m+1)), p = 1..m  (bc > 0 iff cell Peclet < 1);
those of the Kronecker sums are sums mu_p + mu_q (+ mu_r).

All algorithms access A only via products x -> A x.
"""
import numpy as np
import scipy.sparse as sp


def stencil_coeffs(m: int, beta: float):
    """(a, b, c) of the 1D factor T: diagonal, sub-diagonal (u_{i-1}), super (u_{i+1})."""
    ih2 = float((m + 1) * (m + 1))          # 1/h^2
    ih = (m + 1) / 2.0                      # 1/(2h)
    a = 2.0 * ih2
    b = -ih2 - beta * ih
    c = -ih2 + beta * ih
    return a, b, c


def toeplitz_1d(m: int, beta: float):
    a, b, c = stencil_coeffs(m, beta)
    return sp.diags([np.full(m - 1, b), np.full(m, a), np.full(m - 1, c)],
                    [-1, 0, 1], format="csr")


def stencil_matrix(dim: int, m: int, beta: float):
    """A for the 2D (dim=2) or 3D (dim=3) config, as scipy CSR (Kronecker sum)."""
    T = toeplitz_1d(m, beta)
    I = sp.identity(m, format="csr")
    if dim == 1:
        A = T
    elif dim == 2:
        A = (sp.kron(I, T) + sp.kron(T, I)).tocsr()
    elif dim == 3:
        II = sp.identity(m * m, format="csr")
        A = (sp.kron(II, T) + sp.kron(sp.kron(I, T), I) + sp.kron(T, II)).tocsr()
    else:
        raise ValueError(dim)
    A.eliminate_zeros()
    return A


def csr_matrix(row_ptr, col_idx, val, n):
    return sp.csr_matrix((np.asarray(val, dtype=np.float64),
                          np.asarray(col_idx, dtype=np.int64),
                          np.asarray(row_ptr, dtype=np.int64)), shape=(n, n))


def closed_form_eigs_1d(m: int, beta: float):
    a, b, c = stencil_coeffs(m, beta)
    p = np.arange(1, m + 1)
    return a + 2.0 * np.sqrt(b * c) * np.cos(p * np.pi / (m + 1))


def closed_form_eigs(dim: int, m: int, beta: float):
    mu = closed_form_eigs_1d(m, beta)
    if dim == 1:
        return np.sort(mu)
    if dim == 2:
        return np.sort((mu[:, None] + mu[None, :]).ravel())
    return np.sort((mu[:, None, None] + mu[None, :, None] + mu[None, None, :]).ravel())


def spectral_box(dim: int, m: int, beta: float):
    """(c, dx, dy) of an axis-aligned box containing the spectrum of the dim-D operator
    (closed form: Kronecker sum of the 1D tridiagonal Toeplitz factor, eigenvalues
    a + 2 sqrt(bc) cos(p pi/(m+1)); real when bc > 0, on a vertical segment when bc < 0).
    Used for the Chebyshev basis ("the spectrum of A is contained in the
    rectangle [c +- dx, +- dy]")."""
    a, b, c = stencil_coeffs(m, beta)
    cosm = np.cos(np.pi / (m + 1))
    if b * c >= 0.0:
        return dim * a, dim * 2.0 * np.sqrt(b * c) * cosm, 0.0
    return dim * a, 0.0, dim * 2.0 * np.sqrt(-b * c) * cosm
