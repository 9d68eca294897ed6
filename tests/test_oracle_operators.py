"""Pins of oracle/operators.py against what the mathematics fixes.

* coefficients: hand-derived golden values (tests/golden/stencil_coeffs.json);
* consistency: centred differences are EXACT on quadratics, so for every grid
  point whose neighbours are all interior, (A u)(p) = -Lap(u) + beta*grad(u).1
  at p for u = polynomial of degree <= 2 (catches a wrong sign, scale or index);
* spectrum: closed form a + 2 sqrt(bc) cos(p pi/(m+1)) (BASELINE north_star) and
  its Kronecker sums vs LAPACK eigvals of the dense matrix;
* structure of the C4 CSR input (O20).
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from inputs import random_csr_c4

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_golden_coefficients():
    g = json.load(open(os.path.join(GOLD, "stencil_coeffs.json")))
    for name in ("C1", "C2", "C3", "C5"):
        v = g[name]
        a, b, c = O.stencil_coeffs(v["m"], v["beta"])
        assert v["dim"] * a == v["centre"]
        assert b == v["minus"] and c == v["plus"]
    # and the assembled matrix carries them (C1, row of an interior point)
    A = O.stencil_matrix(2, 32, 20.0)
    p = 5 + 32 * 7
    row = A.getrow(p).toarray().ravel()
    assert row[p] == 4356.0
    assert row[p - 1] == -1419.0 and row[p - 32] == -1419.0
    assert row[p + 1] == -759.0 and row[p + 32] == -759.0
    assert np.count_nonzero(row) == 5


@pytest.mark.parametrize("dim,m,beta", [(2, 7, 3.0), (2, 9, 20.0), (3, 5, 4.0), (3, 6, 30.0)])
def test_exact_on_quadratics(dim, m, beta):
    h = 1.0 / (m + 1)
    A = O.stencil_matrix(dim, m, beta)
    grid = np.arange(1, m + 1) * h
    if dim == 2:
        X, Y = np.meshgrid(grid, grid, indexing="xy")   # X varies fastest in ravel
        coords = [X.ravel(), Y.ravel()]
    else:
        Z, Y, X = np.meshgrid(grid, grid, grid, indexing="ij")
        coords = [X.ravel(), Y.ravel(), Z.ravel()]
    # u = sum_a (alpha_a x_a^2 + gamma_a x_a) ; -Lap u = -2 sum alpha ; grad u . 1 = sum(2 alpha x + gamma)
    rng = np.random.default_rng(0)
    alpha = rng.standard_normal(dim)
    gamma = rng.standard_normal(dim)
    u = sum(alpha[a] * coords[a] ** 2 + gamma[a] * coords[a] for a in range(dim))
    Au = A @ u
    expect = -2 * alpha.sum() + beta * sum(2 * alpha[a] * coords[a] + gamma[a] for a in range(dim))
    # interior-of-interior points (no neighbour on the Dirichlet boundary)
    idx = np.arange(m ** dim)
    ii = [idx % m, (idx // m) % m, idx // (m * m)][:dim]
    inner = np.all([(t >= 1) & (t <= m - 2) for t in ii], axis=0)
    np.testing.assert_allclose(Au[inner], expect[inner], rtol=1e-9, atol=1e-7 * np.abs(Au).max())


@pytest.mark.parametrize("dim,m,beta", [(1, 40, 10.0), (2, 10, 8.0), (3, 6, 5.0)])
def test_closed_form_spectrum(dim, m, beta):
    A = O.stencil_matrix(dim, m, beta).toarray()
    ev = np.linalg.eigvals(A)
    assert np.abs(ev.imag).max() < 1e-8 * np.abs(ev).max()
    np.testing.assert_allclose(np.sort(ev.real), O.closed_form_eigs(dim, m, beta), rtol=1e-10)


def test_dirichlet_boundary_rows():
    # corner row of the 2D operator has exactly 3 nonzeros (two neighbours dropped)
    A = O.stencil_matrix(2, 8, 3.0)
    assert A.getrow(0).nnz == 3
    A3 = O.stencil_matrix(3, 5, 3.0)
    assert A3.getrow(0).nnz == 4
    assert A3.getrow(2 + 5 * 2 + 25 * 2).nnz == 7


def test_csr_c4_structure():
    n = 5000
    rp, ci, v, f = random_csr_c4(n, seed=3)
    assert rp.dtype == np.int32 and ci.dtype == np.int32
    assert rp[-1] == 17 * n and f.shape == (n,)
    C = ci.reshape(n, 17)
    V = v.reshape(n, 17)
    assert np.all(np.diff(C, axis=1) > 0)                 # sorted, distinct
    rows = np.arange(n)[:, None]
    diag = C == rows
    assert np.all(diag.sum(axis=1) == 1)
    assert np.all(V[diag] == 6.0)
    off = V[~diag]
    assert abs(off.std() - 0.25) < 0.01 and abs(off.mean()) < 0.01
    # reproducible
    rp2, ci2, v2, f2 = random_csr_c4(n, seed=3)
    assert np.array_equal(ci, ci2) and np.array_equal(v, v2) and np.array_equal(f, f2)
