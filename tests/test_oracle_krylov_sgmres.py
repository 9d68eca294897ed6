"""Pins of oracle/krylov.py and oracle/sgmres.py.

Krylov (Eq. partorth):
* k >= d-1 gives a full Arnoldi basis: ||B^T B - I|| < 1e-12 (d <= 40);
* recurrence identity  A B[:, :d-1] = B Hbar  (definition of the process);
* span(B) = span(full Arnoldi basis) (principal angles) -- both are K_d(A; r);
* each b_j is orthogonal to its k predecessors and has unit norm;
* breakdown on an invariant vector (A = I).
sGMRES (Alg. 1, Eqs. sgmres/sgmres-yhat/sgmres-rhat):
* identity "sketch" S = I reproduces the exact basis-restricted LS (GMRES problem);
* d = n, k = n-1 on a small dense system reproduces the LU solution;
* sandwich (Eq. sgmres-residual) with the MEASURED distortion of S;
* a-posteriori estimate (Eq. sgmres-residual-norm);
* r_est,j nonincreasing in j (nested least-squares problems);
* SPEC worked examples (QR and triangular solve).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.linalg import solve_triangular, subspace_angles

import oracle as O
from oracle.krylov import partial_arnoldi_next
from inputs import rhs_normal

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _c1():
    A = O.stencil_matrix(2, 32, 20.0)
    return A, rhs_normal(1024, 0)


def test_full_orthogonalisation_limit():
    A, f = _c1()
    for d in (20, 40):
        bas = O.partial_arnoldi(lambda v: A @ v, f, d, k=d)
        B = bas["B"]
        assert np.linalg.norm(B.T @ B - np.eye(d), 2) < 1e-12


@pytest.mark.parametrize("k", [1, 2, 4])
def test_recurrence_identity_and_local_orthogonality(k):
    A, f = _c1()
    d = 40
    bas = O.partial_arnoldi(lambda v: A @ v, f, d, k)
    B, M, H = bas["B"], bas["M"], bas["H"]
    # A B_{d-1} = B_d Hbar[:d, :d-1]
    lhs = A @ B[:, :d - 1]
    np.testing.assert_allclose(lhs, M[:, :d - 1], rtol=0, atol=1e-12 * np.abs(lhs).max())
    rhs = B @ H[:d, :d - 1]
    assert np.linalg.norm(lhs - rhs) < 1e-12 * np.linalg.norm(lhs)
    assert np.allclose(np.linalg.norm(B, axis=0), 1.0, atol=1e-14)
    G = B.T @ B
    for j in range(d):
        for i in range(max(0, j - k), j):
            assert abs(G[i, j]) < 1e-12
    # the band: column j-1 of H is nonzero only in rows j-k..j
    for j in range(1, d):
        col = H[:, j - 1]
        nz = np.nonzero(col)[0]
        assert nz.min() >= max(0, j - k) and nz.max() == j


def test_span_equals_full_arnoldi():
    A, f = _c1()
    d = 20
    bas = O.partial_arnoldi(lambda v: A @ v, f, d, k=2)
    Q, _ = O.full_arnoldi(lambda v: A @ v, f, d)
    ang = subspace_angles(bas["B"], Q[:, :d])
    assert ang.max() < 1e-8


def test_breakdown_on_invariant_vector():
    n = 50
    e = np.zeros(n)
    e[3] = 2.0
    bas = O.partial_arnoldi(lambda v: v.copy(), e, 5, 2)
    assert bas["breakdown"] and bas["d_eff"] == 1


def test_spec_worked_examples():
    g = json.load(open(os.path.join(GOLD, "small_linalg.json")))
    U, T = O.thin_qr(np.array(g["qr"]["M"]))
    np.testing.assert_allclose(U, g["qr"]["U"], rtol=1e-15)
    np.testing.assert_allclose(T, g["qr"]["T"], rtol=1e-15)
    y = solve_triangular(np.array(g["trisolve"]["T"]), np.array(g["trisolve"]["b"]))
    np.testing.assert_allclose(y, g["trisolve"]["y"], rtol=1e-15)
    # T diag >= 0 convention on a random matrix, and reconstruction
    rng = np.random.default_rng(0)
    C = rng.standard_normal((64, 16))
    U, T = O.thin_qr(C)
    assert np.all(np.diag(T) >= 0) and np.allclose(np.tril(T, -1), 0)
    assert np.linalg.norm(C - U @ T) < 1e-14 * np.linalg.norm(C)
    assert np.linalg.norm(U.T @ U - np.eye(16)) < 1e-14 * 4


def test_identity_sketch_reproduces_exact_ls():
    A, f = _c1()
    d, k = 30, 2
    n = f.size
    out = O.sgmres_cycle(lambda v: A @ v, f, np.zeros(n), d, k, s=n, zeta=1, seed=0,
                         cycle=0, early_exit_factor=0.0, S=sp.identity(n, format="csr"))
    M = out["basis"]["M"]
    y_exact = O.gmres_exact_ls(M, f)
    np.testing.assert_allclose(out["yhat"], y_exact, rtol=1e-9,
                               atol=1e-10 * np.abs(y_exact).max())
    assert abs(out["r_est"][-1] - np.linalg.norm(f - M @ y_exact)) < 1e-10 * np.linalg.norm(f)


def test_full_dimension_reproduces_lu():
    rng = np.random.default_rng(3)
    n = 50
    A = rng.standard_normal((n, n)) + 10 * np.eye(n)
    f = rng.standard_normal(n)
    res = O.sgmres_solve(lambda v: A @ v, f, d=n, k=n - 1, s=2 * n, zeta=8, seed=9,
                         tol=1e-14, max_cycles=1, early_exit_factor=0.0)
    x = np.linalg.solve(A, f)
    assert np.linalg.norm(res["x"] - x) / np.linalg.norm(x) < 1e-8


def _distortion(S, Bsub):
    Q, _ = np.linalg.qr(Bsub)
    sv = np.linalg.svd(S @ Q, compute_uv=False)
    return max(sv.max() - 1, 1 - sv.min())


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_sandwich_and_estimate(seed):
    A, f = _c1()
    n = f.size
    d, k, s, z = 50, 2, 100, 8
    S = O.sketch_matrix(n, s, z, seed=seed)
    out = O.sgmres_cycle(lambda v: A @ v, f, np.zeros(n), d, k, s, z, seed, 0,
                         early_exit_factor=0.0, S=S)
    M = out["basis"]["M"]
    eps = _distortion(S, np.column_stack([M, f]))
    assert eps < 1
    y_star = O.gmres_exact_ls(M, f)
    r_gm = np.linalg.norm(M @ y_star - f)
    r_sg = np.linalg.norm(A @ out["x"] - f)
    assert r_gm <= r_sg * (1 + 1e-10)
    assert r_sg <= (1 + eps) / (1 - eps) * r_gm
    ratio = out["r_est"][-1] / r_sg
    assert (1 - eps) - 1e-9 <= ratio <= (1 + eps) + 1e-9
    # nested least squares: r_est,j is nonincreasing
    assert np.all(np.diff(out["r_est"]) <= 1e-12 * out["r_est"][0])


def test_restarted_c1_converges():
    A, f = _c1()
    res = O.sgmres_solve(lambda v: A @ v, f, 60, 2, 120, 8, 0, tol=1e-8, max_cycles=4)
    assert res["rel_res_true"] <= 1e-8 and res["cycles"] <= 3
    assert np.all(np.diff(res["hist_true"]) < 0)
    # early exit (O16) stopped the last cycle before d columns
    assert res["columns"] < 60 * res["cycles"]


def test_partial_arnoldi_next_column_matches():
    A, f = _c1()
    bas = O.partial_arnoldi(lambda v: A @ v, f, 21, 2)
    bas20 = O.partial_arnoldi(lambda v: A @ v, f, 20, 2)
    b, h, nu = partial_arnoldi_next(lambda v: A @ v, bas20["B"], bas20["M"], 2)
    np.testing.assert_allclose(b, bas["B"][:, 20], atol=1e-15)
    np.testing.assert_allclose(h, bas["H"][:20, 19], atol=1e-9)
    assert abs(nu - bas["H"][20, 19]) < 1e-9
