"""Pins of oracle/srr.py (Alg. 2).

* closed-form eigenvalues (BASELINE north_star): 1D tridiagonal-Toeplitz
  convection-diffusion, d = n (the basis spans R^n), Ritz values = a + 2 sqrt(bc) cos(p pi/(n+1));
* Krylov identity: Mhat and the Arnoldi-type recurrence matrix
  "differ only in the final column": Mhat[:, :d-1] = Hbar[:d, :d-1];
* similarity invariance B <- B G;
* a-posteriori bound Eq. rescompare with the measured distortion;
* canonical ordering of conjugate pairs (reading O23).
"""
import numpy as np
import pytest

import oracle as O
from inputs import rhs_normal
from oracle.srr import srr_from_basis


@pytest.mark.parametrize("n,beta", [(64, 5.0), (100, 10.0)])
def test_closed_form_eigenvalues_full_dimension(n, beta):
    A = O.stencil_matrix(1, n, beta)
    v0 = rhs_normal(n, 4)
    out = O.srr_eigs(lambda v: A @ v, v0, d=n, k=n, s=2 * n, zeta=8, seed=4, nev=n)
    th = np.sort(out["theta"].real)
    assert np.abs(out["theta"].imag).max() < 1e-8 * np.abs(th).max()
    np.testing.assert_allclose(th, np.sort(O.closed_form_eigs_1d(n, beta)), rtol=1e-9)


def test_krylov_identity_final_column():
    A = O.stencil_matrix(2, 32, 10.0)
    v0 = rhs_normal(1024, 4)
    d = 40
    out = O.srr_eigs(lambda v: A @ v, v0, d=d, k=2, s=2 * d, zeta=8, seed=4, nev=10)
    H = out["basis"]["H"]
    Mh = out["Mhat"]
    scale = np.abs(Mh).max()
    assert np.abs(Mh[:, :d - 1] - H[:d, :d - 1]).max() < 1e-11 * scale
    assert np.abs(Mh[:, d - 1] - H[:d, d - 1]).max() > 1e-8 * scale   # last column differs


def test_similarity_invariance_and_residual_bound():
    A = O.stencil_matrix(2, 24, 10.0)
    n = 24 * 24
    v0 = rhs_normal(n, 4)
    d, s = 30, 60
    bas = O.partial_arnoldi(lambda v: A @ v, v0, d, 2)
    S = O.sketch_matrix(n, s, 8, seed=4)
    a = srr_from_basis(lambda v: A @ v, bas["B"], bas["M"], S, 6)
    G = np.random.default_rng(1).standard_normal((d, d)) + 4 * np.eye(d)
    b = srr_from_basis(lambda v: A @ v, bas["B"] @ G, bas["M"] @ G, S, 6)
    np.testing.assert_allclose(b["theta"], a["theta"], rtol=1e-8)
    # Eq. rescompare with measured eps on range([B, AB])
    Q, _ = np.linalg.qr(np.column_stack([bas["B"], bas["M"]]))
    sv = np.linalg.svd(S @ Q, compute_uv=False)
    eps = max(sv.max() - 1, 1 - sv.min())
    assert eps < 1
    lo, hi = (1 - eps) / (1 + eps), (1 + eps) / (1 - eps)
    ratio = a["res_true"] / a["res_est"]
    assert np.all(ratio >= lo - 1e-9) and np.all(ratio <= hi + 1e-9)


def test_select_ritz_canonical_order():
    th = np.array([3 + 0j, 1 + 4j, 1 - 4j, -5 + 0j, 0.5 + 0j, 2 + 2j, 2 - 2j])
    sel = O.select_ritz(th, 3)
    # |.|: 5, sqrt17, sqrt17, 3, 2.83, 2.83, .5 -> -5, 1+4j, 1-4j
    assert list(th[sel]) == [-5 + 0j, 1 + 4j, 1 - 4j]
    sel = O.select_ritz(th, 2)
    # position 2 splits the pair 1+-4j -> partner added
    assert list(th[sel]) == [-5 + 0j, 1 + 4j, 1 - 4j]
