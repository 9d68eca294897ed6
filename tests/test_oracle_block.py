"""Pins of oracle.block_chebyshev_basis and oracle.srr_eigs_block (block Krylov for sRR;
Sec. "Block Krylov subspaces" P:1867-1896, "Block Chebyshev recurrence" P:1983-2008).

* closed form: on a diagonal A with a real spectrum (dy = 0) block j is phi_j(A) Omega with
  phi_j(lambda) = 2^-(j-1) T_{j-1}((lambda - c)/rho), T the Chebyshev polynomials of the first kind (numpy's
  Chebyshev series, independent of the recurrence);
* block size 1 reproduces the single-vector Chebyshev basis (oracle.chebyshev_basis, pinned separately), up to the
  start vector's norm;
* the three-term identity A B_1 = 2 rho B_2 + c B_1, A B_j = rho B_{j+1} + c B_j + e B_{j-1} (the relation the GPU
  forms S A B through, reading O34) holds for the explicit products M = A B;
* span(B) = K_p(A; Omega): principal angles against an orthonormalised block monomial basis;
* sRR on a block basis spanning the whole space of a diagonal A (d = b p = n) returns A's eigenvalues exactly
  (they are known: the diagonal);
* sRR with the block basis on the C5 operator at small size: the top Ritz value approaches the closed-form largest
  eigenvalue as the depth p grows (Krylov convergence).
"""
import numpy as np
from numpy.polynomial import chebyshev as Ch
from scipy.linalg import subspace_angles

import oracle as O
from inputs import start_block


def test_closed_form_on_diagonal_operator():
    rng = np.random.default_rng(11)
    lam = np.sort(rng.uniform(2.0, 10.0, 200))
    c, dx = 6.0, 4.0
    Om = rng.standard_normal((200, 5))
    p = 9
    bas = O.block_chebyshev_basis(lambda v: lam * v, Om, p, c, dx, 0.0)
    X = (lam - c) / dx
    for j in range(1, p + 1):
        coef = np.zeros(j)
        coef[j - 1] = 1.0
        ref = (2.0 ** (-(j - 1)) * Ch.chebval(X, coef))[:, None] * Om
        got = bas["B"][:, (j - 1) * 5:j * 5]
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max(), j


def test_block_size_one_is_the_chebyshev_basis():
    A = O.stencil_matrix(2, 24, 15.0)
    box = O.spectral_box(2, 24, 15.0)
    w = start_block(A.shape[0], 1, 9)
    blk = O.block_chebyshev_basis(lambda v: A @ v, w, 12, *box)
    one = O.chebyshev_basis(lambda v: A @ v, w[:, 0], 12, *box)
    ref = one["raw"] * np.linalg.norm(w)
    assert np.abs(blk["B"] - ref).max() <= 1e-13 * np.abs(ref).max()


def test_three_term_identity():
    A = O.stencil_matrix(2, 20, 12.0)
    c, dx, dy = O.spectral_box(2, 20, 12.0)
    rho = max(dx, dy)
    e = (dx * dx - dy * dy) / (4 * rho)
    b, p = 4, 6
    bas = O.block_chebyshev_basis(lambda v: A @ v, start_block(400, b, 2), p, c, dx, dy)
    B, M = bas["B"], bas["M"]
    blk = lambda j: B[:, (j - 1) * b:j * b]  # noqa: E731
    ablk = lambda j: M[:, (j - 1) * b:j * b]  # noqa: E731
    scale = np.abs(M).max()
    assert np.abs(ablk(1) - (2 * rho * blk(2) + c * blk(1))).max() <= 1e-12 * scale
    for j in range(2, p):
        assert np.abs(ablk(j) - (rho * blk(j + 1) + c * blk(j) + e * blk(j - 1))).max() <= 1e-12 * scale


def test_span_is_the_block_krylov_space():
    A = O.stencil_matrix(2, 16, 8.0)
    box = O.spectral_box(2, 16, 8.0)
    b, p = 3, 4
    Om = start_block(256, b, 5)
    bas = O.block_chebyshev_basis(lambda v: A @ v, Om, p, *box)
    K = [Om]
    for _ in range(p - 1):
        K.append(A @ K[-1])
    Q, _ = np.linalg.qr(np.concatenate(K, axis=1))
    Qb, _ = np.linalg.qr(bas["B"])
    assert subspace_angles(Qb, Q).max() <= 1e-8


def test_srr_block_exact_on_the_whole_space():
    rng = np.random.default_rng(4)
    n = 48
    lam = np.sort(rng.uniform(2.0, 10.0, n))
    b, p = 8, 6                                    # d = 48 = n
    out = O.srr_eigs_block(lambda v: lam * v, rng.standard_normal((n, b)), p, 6.0, 4.0, 0.0, 2 * n, 8, 3, 5)
    top = np.sort(lam)[::-1][:5]
    np.testing.assert_allclose(np.sort(out["theta"].real)[::-1], top, rtol=1e-8)
    assert np.abs(out["theta"].imag).max() <= 1e-8 * top[0]
    assert out["res_true"].max() <= 1e-6 * top[0]


def test_srr_block_converges_to_the_top_eigenvalue():
    m, beta = 32, 10.0
    A = O.stencil_matrix(2, m, beta)
    box = O.spectral_box(2, m, beta)
    lam_max = O.closed_form_eigs(2, m, beta).max()
    errs = []
    for p in (2, 4, 8):
        b = 8
        out = O.srr_eigs_block(lambda v: A @ v, start_block(m * m, b, 4), p, *box, 2 * b * p, 8, 4, 1)
        errs.append(abs(out["theta"][0].real - lam_max) / lam_max)
    assert errs[2] < errs[1] < errs[0] and errs[2] < 2e-2, errs
