"""Pins of the oracle's adaptive restarting (Sec. adaptive-restart):
"When first kappa_2(T_j) > tol ... we generate the new Krylov subspace using the previous
residual r_{j-1} = r_0 - AB_{j-1} y_{j-1}".

  * kappa_2(T_j) = kappa_2(SAB_j) (SAB_j = U_j T_j with orthonormal U_j), checked with scipy's SVD of the
    sketched matrix itself, not the QR factor the oracle uses: the chosen j satisfies
    kappa(SAB_j) <= tol < kappa(SAB_{j+1});
  * kappa_2 of the leading blocks is non-decreasing in j (singular-value interlacing) -- the property
    the device's batch check + bisection relies on (reading O31);
  * the adapted cycle's solution is exactly the plain cycle with d = j columns (same S, same basis);
  * a k = 1 basis (condition growing ~2.3x per column) with adaptive restarting still converges to 1e-8.
"""
import numpy as np
from scipy.linalg import svdvals

import oracle as O
from inputs import rhs_normal

M_, BETA, D, K, S_ = 32, 20.0, 40, 1, 80


def _setup():
    A = O.stencil_matrix(2, M_, BETA)
    f = rhs_normal(M_ * M_, 0)
    return A, f


def _kappa(C, j):
    sv = svdvals(C[:, :j])
    return sv[0] / sv[-1]


def test_kappa_of_leading_blocks_is_monotone():
    A, f = _setup()
    out = O.sgmres_cycle(lambda v: A @ v, f, np.zeros_like(f), D, K, S_, 8, 0, 0, early_exit_factor=0.0)
    ks = [_kappa(out["C"], j) for j in range(1, D + 1)]
    assert all(ks[i + 1] >= ks[i] * (1 - 1e-10) for i in range(D - 1))
    assert ks[-1] > 1e9 and ks[0] == 1.0


def test_adaptive_cycle_stops_before_the_threshold():
    A, f = _setup()
    for tol_k in (1e4, 1e6, 3e7):
        out = O.sgmres_cycle(lambda v: A @ v, f, np.zeros_like(f), D, K, S_, 8, 0, 0, early_exit_factor=0.0,
                             cond_tol=tol_k, adaptive=True)
        j = out["j"]
        assert out["flags"] & O.INFO_ADAPTIVE
        assert _kappa(out["C"], j) <= tol_k < _kappa(out["C"], j + 1)


def test_adaptive_solution_is_the_truncated_cycle():
    A, f = _setup()
    x0 = np.zeros_like(f)
    ad = O.sgmres_cycle(lambda v: A @ v, f, x0, D, K, S_, 8, 0, 0, early_exit_factor=0.0, cond_tol=1e6,
                        adaptive=True)
    plain = O.sgmres_cycle(lambda v: A @ v, f, x0, ad["j"], K, S_, 8, 0, 0, early_exit_factor=0.0)
    assert plain["j"] == ad["j"]
    np.testing.assert_allclose(ad["x"], plain["x"], rtol=0, atol=1e-12 * np.abs(plain["x"]).max())


def test_adaptive_solve_converges():
    A, f = _setup()
    res = O.sgmres_solve(lambda v: A @ v, f, D, K, S_, 8, 0, tol=1e-8, max_cycles=40, cond_tol=1e6, adaptive=True)
    assert res["rel_res_true"] <= 1e-8 and res["flags"] & O.INFO_ADAPTIVE
