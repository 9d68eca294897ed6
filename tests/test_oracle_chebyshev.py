"""Pins of oracle.chebyshev_basis (Eq. Chebrecurse) and
oracle.spectral_box.

* closed form: for a real spectrum (dy = 0) the raw recurrence vectors are
  raw_i = 2^-i T_i((A - cI)/rho) raw_0 (Chebyshev polynomials of the first kind, i >= 1),
  checked on a diagonal operator against numpy's Chebyshev series evaluation;
* recurrence identity A B[:, :d-1] = B H[:d, :d-1] (the relation sGMRES/sRR sketch through);
* span(B) = K_d(A; r) (principal angles against the full-Arnoldi basis);
* conditioning grows slowly (polynomially, not exponentially): kappa(B) of the
  normalised Chebyshev basis vs the normalised monomial basis;
* the spectral box of the convection-diffusion operators is the closed-form spectrum's hull;
* sGMRES with the Chebyshev basis solves the same least-squares problem over the same Krylov
  space: restarted C1 reaches 1e-8 and matches the Arnoldi-basis solution.
"""
import numpy as np
from numpy.polynomial import chebyshev as Ch
from scipy.linalg import subspace_angles

import oracle as O
from inputs import rhs_normal


def test_closed_form_on_diagonal_operator():
    rng = np.random.default_rng(3)
    lam = np.sort(rng.uniform(2.0, 10.0, 300))
    c, dx = 6.0, 4.0
    r = rng.standard_normal(300)
    d = 25
    bas = O.chebyshev_basis(lambda v: lam * v, r, d, c, dx, 0.0)
    X = (lam - c) / dx
    raw0 = r / np.linalg.norm(r)
    for i in range(1, d):
        coef = np.zeros(i + 1)
        coef[i] = 1.0
        ref = 2.0 ** (-i) * Ch.chebval(X, coef) * raw0
        assert np.abs(bas["raw"][:, i] - ref).max() <= 1e-13 * max(np.abs(ref).max(), 1e-300), i
    assert np.allclose(np.linalg.norm(bas["B"], axis=0), 1.0, rtol=0, atol=1e-14)


def test_recurrence_identity_and_span():
    A = O.stencil_matrix(2, 32, 20.0)
    f = rhs_normal(1024, 0)
    box = O.spectral_box(2, 32, 20.0)
    d = 30
    bas = O.chebyshev_basis(lambda v: A @ v, f, d, *box)
    B, H = bas["B"], bas["H"]
    lhs = A @ B[:, :d - 1]
    assert np.abs(lhs - B @ H[:d, :d - 1]).max() <= 1e-13 * np.abs(lhs).max()
    np.testing.assert_allclose(bas["M"], A @ B, rtol=0, atol=1e-12 * np.abs(A @ B).max())
    Q, _ = O.full_arnoldi(lambda v: A @ v, f, 10)
    ang = subspace_angles(B[:, :10], Q[:, :10])
    assert ang.max() <= 1e-8


def test_conditioning_grows_slowly():
    A = O.stencil_matrix(2, 32, 20.0)
    f = rhs_normal(1024, 0)
    box = O.spectral_box(2, 32, 20.0)
    d = 40
    bas = O.chebyshev_basis(lambda v: A @ v, f, d, *box)
    mono = np.zeros((1024, d))
    mono[:, 0] = f / np.linalg.norm(f)
    for j in range(1, d):
        v = A @ mono[:, j - 1]
        mono[:, j] = v / np.linalg.norm(v)
    assert np.linalg.cond(bas["B"]) < 1e2 and np.linalg.cond(mono) > 1e12


def test_spectral_box_is_the_spectrum_hull():
    for dim, m, beta in [(2, 32, 20.0), (3, 12, 10.0), (2, 16, 5.0), (3, 160, 30.0)]:
        c, dx, dy = O.spectral_box(dim, m, beta)
        ev = O.closed_form_eigs(dim, m, beta)
        assert dy == 0.0
        np.testing.assert_allclose([c - dx, c + dx], [ev.min(), ev.max()], rtol=1e-13)
    # cell Peclet > 1: the 1D factor's eigenvalues are complex, on the vertical segment Re = a
    c, dx, dy = O.spectral_box(1, 8, 500.0)
    a, b, cc = O.stencil_coeffs(8, 500.0)
    assert b * cc < 0 and dx == 0.0 and c == a and dy > 0.0


def test_sgmres_chebyshev_matches_arnoldi_space():
    A = O.stencil_matrix(2, 32, 20.0)
    f = rhs_normal(1024, 0)
    box = O.spectral_box(2, 32, 20.0)
    rc = O.sgmres_solve(lambda v: A @ v, f, 60, 2, 120, 8, 0, tol=1e-8, max_cycles=10, cheb=box)
    ra = O.sgmres_solve(lambda v: A @ v, f, 60, 2, 120, 8, 0, tol=1e-8, max_cycles=10)
    assert rc["rel_res_true"] <= 1e-8 and rc["cycles"] == ra["cycles"]
    np.testing.assert_allclose(rc["x"], ra["x"], rtol=0, atol=1e-6 * np.abs(ra["x"]).max())
