"""Pins of oracle.whitened_basis / sgmres_cycle(whiten=True): whitening instead of restarting (
Fact "Whitening" P:598-612, Sec. "Adaptive restarting" P:1398-1400; reading O36).

* the Fact itself: at every whitening event the whitened reduced matrix A B_J T_J^{-1} has
  kappa_2 <= (1 + eps)/(1 - eps), eps the distortion of S on range(A B_J) measured by an SVD (eq:whitening), and its
  sketch S A B_J T_J^{-1} is orthonormal (= U_J);
* whitening changes the basis, never the nested Krylov spaces: span of the first j columns = K_j(A; r) (principal
  angles against full Arnoldi), so the sGMRES iterate and every r_est,j equal those of the plain k-truncated basis
  with the same number of columns (sGMRES depends only on the subspace and S);
* every basis vector has unit norm;
* generation stops (with the columns so far) when the threshold is crossed again without progress;
* restarted whitened sGMRES reaches 1e-8 on C1.
"""
import numpy as np
from scipy.linalg import subspace_angles

import oracle as O
from inputs import rhs_normal


def _c1():
    A = O.stencil_matrix(2, 32, 20.0)
    return (lambda v: A @ v), A, rhs_normal(1024, 0), O.sketch_matrix(1024, 120, 8, 0, 0)


def test_fact_whitening_at_every_event():
    mv, A, f, S = _c1()
    b = O.whitened_basis(mv, f, 60, 2, S, 100.0, record=True)
    assert len(b["snapshots"]) >= 3
    for J, Mw in b["snapshots"]:
        Q, _ = np.linalg.qr(Mw)
        sv = np.linalg.svd(S @ Q, compute_uv=False)
        eps = max(sv[0] - 1.0, 1.0 - sv[-1])
        assert eps < 1.0
        assert np.linalg.cond(Mw) <= (1 + eps) / (1 - eps) * (1 + 1e-10), (J, np.linalg.cond(Mw), eps)
        G = (S @ Mw).T @ (S @ Mw)
        assert np.abs(G - np.eye(J)).max() <= 1e-10


def test_same_krylov_spaces_and_same_iterate():
    mv, A, f, S = _c1()
    b = O.whitened_basis(mv, f, 60, 2, S, 100.0)
    B = b["B"]
    assert np.allclose(np.linalg.norm(B, axis=0), 1.0, atol=1e-13)
    Q, _ = O.full_arnoldi(mv, f, 40)
    for j in (5, 20, 35):
        assert subspace_angles(B[:, :j], Q[:, :j]).max() <= 1e-8
    de = b["d_eff"]
    w = O.sgmres_cycle(mv, f, np.zeros(1024), 60, 2, 120, 8, 0, 0, early_exit_factor=0, cond_tol=100.0, whiten=True)
    p = O.sgmres_cycle(mv, f, np.zeros(1024), de, 2, 120, 8, 0, 0, early_exit_factor=0)
    assert w["j"] == de and w["flags"] & O.INFO_WHITEN
    assert np.abs(w["x"] - p["x"]).max() <= 1e-10 * np.abs(p["x"]).max()
    np.testing.assert_allclose(w["r_est"], p["r_est"], rtol=1e-10)


def test_stops_without_progress():
    mv, A, f, S = _c1()
    b = O.whitened_basis(mv, f, 60, 2, S, 10.0)
    assert b["stopped"] and b["d_eff"] < 60 and b["d_eff"] == b["events"][-1]


def test_restarted_whitened_sgmres_converges():
    mv, A, f, S = _c1()
    res = O.sgmres_solve(mv, f, 60, 2, 120, 8, 0, tol=1e-8, max_cycles=10, cond_tol=100.0, whiten=True)
    assert res["rel_res_true"] <= 1e-8 and res["flags"] & O.INFO_WHITEN
    assert np.linalg.norm(f - A @ res["x"]) / np.linalg.norm(f) <= 1e-8
