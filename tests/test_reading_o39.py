"""Pins of reading O39: the forms the default 3D step kernel uses instead of a second stencil.

* forward-edge quadratic form: <w, A w> = cc ||w||^2 + (cm + cp) sum_p w_p (w_{p+x} + w_{p+y} [+ w_{p+z}]) for the
  centred-difference operator with zero Dirichlet values outside (each grid edge (p, p+e) contributes
  w_p cp w_{p+e} from row p and w_{p+e} cm w_p from row p+e), checked against the oracle's Kronecker-sum matrix;
* transposed dot: <U, A w> = <A^T U, w> with A^T the same stencil with cm and cp swapped;
* derived breakdown reference: in k-truncated Arnoldi (Eq. partorth) every k+1 consecutive columns are
  orthonormal, so m_{j-1} = w_j + sum_l Hbar[l, j-1] b_l gives ||m_{j-1}||^2 = ||w_j||^2 + sum_l Hbar[l, j-1]^2,
  checked on the oracle's own basis.
Nothing here imports the CUDA path.
"""
import numpy as np
import pytest

import oracle as O


def _fe_form(w, dim, m, cc, cm, cp):
    g = w.reshape((m,) * dim)  # C order: the last axis is x (contiguous), as in the library's layout
    e = 0.0
    for ax in range(dim):
        a = np.swapaxes(g, ax, -1)
        e += float(np.sum(a[..., :-1] * a[..., 1:]))
    return cc * float(w @ w) + (cm + cp) * e


@pytest.mark.parametrize("dim,m,beta", [(2, 9, 20.0), (2, 12, 50.0), (3, 6, 30.0), (3, 7, 0.0)])
def test_forward_edge_quadratic_form(dim, m, beta):
    A = O.stencil_matrix(dim, m, beta)
    a, b, c = O.stencil_coeffs(m, beta)
    cc, cm, cp = dim * a, b, c
    rng = np.random.default_rng(dim * 100 + m)
    for _ in range(3):
        w = rng.standard_normal(m ** dim)
        ref = float(w @ (A @ w))
        got = _fe_form(w, dim, m, cc, cm, cp)
        assert abs(got - ref) <= 1e-12 * cc * float(w @ w)
    # a smooth vector (strong cancellation between the two terms) still agrees to rounding
    x = np.linspace(0, 1, m + 2)[1:-1]
    grids = np.meshgrid(*([x] * dim), indexing="ij")
    w = np.prod([np.sin(np.pi * t) for t in grids], axis=0).ravel()
    assert abs(_fe_form(w, dim, m, cc, cm, cp) - float(w @ (A @ w))) <= 1e-12 * cc * float(w @ w)


@pytest.mark.parametrize("dim,m,beta", [(2, 10, 20.0), (3, 6, 30.0)])
def test_transposed_dot(dim, m, beta):
    A = O.stencil_matrix(dim, m, beta)
    At = O.stencil_matrix(dim, m, -beta)  # swapping cm and cp = reversing the convection
    assert abs(At - A.T).max() == 0.0
    rng = np.random.default_rng(7)
    u, w = rng.standard_normal((2, m ** dim))
    assert abs(float(u @ (A @ w)) - float((At @ u) @ w)) <= 1e-12 * np.linalg.norm(A @ w) * np.linalg.norm(u)


@pytest.mark.parametrize("k", [1, 2, 4])
def test_derived_breakdown_reference(k):
    A = O.stencil_matrix(2, 16, 20.0)
    r = np.random.default_rng(3).standard_normal(A.shape[0])
    res = O.partial_arnoldi(lambda v: A @ v, r, 40, k)
    B, M, H = res["B"], res["M"], res["H"]
    d = res["d_eff"]
    for j in range(1, d):
        lo = max(0, j - k)
        # orthonormal window of k+1 consecutive columns
        Wn = B[:, lo:j + 1]
        assert np.abs(Wn.T @ Wn - np.eye(j + 1 - lo)).max() < 1e-12
        m = M[:, j - 1]
        derived = np.sqrt(H[j, j - 1] ** 2 + np.sum(H[lo:j, j - 1] ** 2))
        assert abs(derived - np.linalg.norm(m)) <= 1e-13 * np.linalg.norm(m)
