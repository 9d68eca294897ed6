"""Pins of the oracle's stabilised sRR (Sec. "Stabilization"; reading O33), against facts
that do not come from the implementation:

  * an exactly rank-deficient basis spanning an invariant subspace of a diagonal A: the truncated-SVD
    pencil returns the subspace's eigenvalues exactly (closed form), with zero residuals, although
    T is numerically singular (the unstabilised Mhat = T^-1 U^T D is meaningless there);
  * without truncation (well-conditioned basis, r = d) the pencil is similar to Mhat, so its
    eigenvalues equal the unstabilised sRR's (pinned by tests/test_oracle_srr.py);
  * "if_ill" switches exactly when kappa_2(T) exceeds tol (Alg. 2);
  * every returned pair solves the r x r generalized problem (U^T D V) z = theta Sigma z (QZ
    residual), and r counts the singular values >= sigma_1 / tol;
  * on a Krylov basis with kappa_2(T) ~ 1e17 (k = 1) the stabilised Ritz values approach A's
    dominant eigenvalues (dense eig) while the unstabilised ones do not.
"""
import numpy as np
import scipy.sparse as sp

import oracle as O
from inputs import start_vector


def test_invariant_subspace_rank_deficient_basis_gives_exact_eigenvalues():
    rng = np.random.default_rng(11)
    n, r, d, s = 300, 6, 20, 60
    lam = np.linspace(1.0, 50.0, n)[::-1].copy()           # distinct, largest first
    A = sp.diags(lam)
    idx = rng.choice(n, r, replace=False)
    E = np.zeros((n, r))
    E[idx, np.arange(r)] = 1.0
    Q, _ = np.linalg.qr(E @ rng.standard_normal((r, r)))   # an invariant subspace, mixed basis
    B = np.hstack([Q, Q @ rng.standard_normal((r, d - r))])  # rank r exactly
    M = A @ B
    S = O.sketch_matrix(n, s, 8, 3, 0)
    out = O.srr_from_basis(lambda x: A @ x, B, M, S, r, stabilize="always", tol=1e10)
    assert out["stabilized"] and out["rank"] == r
    np.testing.assert_allclose(np.sort(out["theta"].real), np.sort(lam[idx]), rtol=1e-10)
    assert np.abs(out["theta"].imag).max() <= 1e-10 * lam.max()
    assert out["res_true"].max() <= 1e-9 * lam.max()
    assert np.linalg.cond(out["T"]) > 1e12                 # the unstabilised problem is singular


def test_no_truncation_matches_unstabilised_srr():
    m, beta, d = 16, 5.0, 30
    n = m * m
    Ao = O.stencil_matrix(2, m, beta)
    v0 = start_vector(n, 4)
    a = O.srr_eigs(lambda x: Ao @ x, v0, d, 2, 2 * d, 8, 4, 8)
    b = O.srr_eigs(lambda x: Ao @ x, v0, d, 2, 2 * d, 8, 4, 8, stabilize="always", tol=1e14)
    assert not a["stabilized"] and b["stabilized"] and b["rank"] == d
    ta, tb = a["theta_all"], b["theta_all"]                # same multiset (nearest match both ways)
    assert max(np.abs(tb - t).min() for t in ta) <= 1e-11 * np.abs(ta).max()
    assert max(np.abs(ta - t).min() for t in tb) <= 1e-11 * np.abs(ta).max()
    np.testing.assert_allclose(np.sort(b["res_true"]), np.sort(a["res_true"]), rtol=1e-6)


def test_if_ill_switch_and_pencil_residual():
    m, beta = 24, 10.0
    n = m * m
    Ao = O.stencil_matrix(2, m, beta)
    v0 = start_vector(n, 4)
    d, k, s, tol = 200, 1, 420, 1e8
    well = O.srr_eigs(lambda x: Ao @ x, v0, 30, 2, 60, 8, 4, 4, stabilize="if_ill", tol=tol)
    assert not well["stabilized"] and np.linalg.cond(well["T"]) < tol
    ill = O.srr_eigs(lambda x: Ao @ x, v0, d, k, s, 8, 4, 4, stabilize="if_ill", tol=tol)
    assert ill["stabilized"] and np.linalg.cond(ill["T"]) > tol
    sig = ill["sigma"]
    r = ill["rank"]
    assert r == np.count_nonzero(sig >= sig[0] / tol) and r < d
    Uc, _, Vh = np.linalg.svd(ill["C"], full_matrices=False)
    A_r = Uc[:, :r].T @ ill["D"] @ Vh[:r].T
    Z = Vh[:r] @ ill["Y"]                                  # y = V_r z  ->  z = V_r^T y
    scale = np.linalg.norm(A_r, 2)
    for t, z in zip(ill["theta"], Z.T):                    # QZ is backward stable: residual ~ u (|A_r| + |t| |Sigma|)
        res = np.linalg.norm(A_r @ z - t * (sig[:r] * z))
        assert res <= 1e-12 * (scale + abs(t) * sig[0]) * np.linalg.norm(z)


def test_stabilised_ritz_values_approach_dominant_eigenvalues():
    m, beta = 24, 10.0
    n = m * m
    Ao = O.stencil_matrix(2, m, beta)
    v0 = start_vector(n, 4)
    ev = np.linalg.eigvals(Ao.toarray())
    lam1 = ev[np.argmax(np.abs(ev))]
    plain = O.srr_eigs(lambda x: Ao @ x, v0, 200, 1, 420, 8, 4, 2)
    stab = O.srr_eigs(lambda x: Ao @ x, v0, 200, 1, 420, 8, 4, 2, stabilize="always", tol=1e8)
    assert abs(stab["theta"][0] - lam1) <= 1e-5 * abs(lam1)
    assert stab["res_true"][0] <= 1e-5 * abs(lam1)
    assert plain["res_true"][0] >= 1e-2 * abs(lam1)        # k = 1, kappa ~ 1e17: plain sRR fails
