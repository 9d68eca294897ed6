"""GPU edge cases through the C-ABI (-m gpu), each against the oracle or a closed form:

  * argument errors come back as SKS_EINVAL (sks.h): sizes outside the header's
    ranges, a non-finite right-hand side, bad nev;
  * the degenerate inputs of the method: a zero right-hand side (x = 0 exactly), a lucky breakdown
    on an exact eigenvector of A (reading O10: the basis stops, x = f / lambda), an sRR start vector
    that spans an invariant subspace (fewer than 2 columns: SKS_EINVAL), a single basis column
    (d = 1), full orthogonalisation k >= d (orthonormal basis, Eq. partorth with the whole window);
  * the smallest stencil (m = 2) and the largest window (k = 8).
"""
import numpy as np
import pytest

import oracle as O
from inputs import rhs_normal, start_vector

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200 import build
    build.build()
    c = P.Context(0)
    yield c
    c.close()


def _P():
    import paper_2111_00113_b200 as P
    return P


def _eigvec_2d(m, beta, p=1):
    """Closed-form eigenvector of the 2D operator (Kronecker sum of the 1D factor T = tridiag(b, a, c),
    b, c < 0): u_i = (b/c)^(i/2) sin(i p pi/(m+1)), T u = (a - 2 sqrt(bc) cos(p pi/(m+1))) u;
    A (u x u) = 2 lambda (u x u)."""
    a, b, c = O.stencil_coeffs(m, beta)
    i = np.arange(1, m + 1)
    u = (b / c) ** (i / 2.0) * np.sin(i * p * np.pi / (m + 1))
    lam = a - 2.0 * np.sqrt(b * c) * np.cos(p * np.pi / (m + 1))
    f = np.outer(u, u).ravel()
    return f / np.linalg.norm(f), 2.0 * lam


BAD_SGMRES = [dict(d=0), dict(s=20), dict(s=4096), dict(zeta=0), dict(zeta=17), dict(k=0), dict(k=9),
              dict(tol=-1.0), dict(max_cycles=0)]


@pytest.mark.parametrize("bad", BAD_SGMRES)
def test_sgmres_rejects_bad_arguments(ctx, bad):
    P = _P()
    kw = dict(d=20, k=2, s=40, zeta=8, seed=0, tol=1e-8, max_cycles=2)
    kw.update(bad)
    with pytest.raises(P.SksError) as e:
        ctx.sgmres_solve(P.StencilOperator(2, 16, 5.0), rhs_normal(256, 0), **kw)
    assert e.value.status == -1 and "SKS_EINVAL" in str(e.value)


def test_sgmres_rejects_non_finite_rhs(ctx):
    P = _P()
    f = rhs_normal(256, 0)
    f[17] = np.nan
    with pytest.raises(P.SksError) as e:
        ctx.sgmres_solve(P.StencilOperator(2, 16, 5.0), f, d=20, k=2, s=40)
    assert e.value.status == -1


@pytest.mark.parametrize("nev,d", [(0, 20), (12, 40), (5, 1)])
def test_srr_rejects_bad_arguments(ctx, nev, d):
    P = _P()
    with pytest.raises(P.SksError) as e:
        ctx.srr_eigs(P.StencilOperator(2, 16, 5.0), start_vector(256, 4), d=d, k=2, s=2 * d + 2, nev=nev)
    assert e.value.status == -1


def test_stencil_rejects_m_below_2(ctx):
    P = _P()
    with pytest.raises(P.SksError):
        ctx.sgmres_solve(P.StencilOperator(2, 1, 5.0), np.ones(1), d=1, k=1, s=2)


def test_sgmres_zero_rhs_gives_zero(ctx):
    P = _P()
    res = ctx.sgmres_solve(P.StencilOperator(2, 16, 5.0), np.zeros(256), d=20, k=2, s=40, max_cycles=3)
    assert res.converged and np.all(res.x == 0.0)


@pytest.mark.parametrize("dim", [2, 3])
def test_sgmres_lucky_breakdown_on_eigenvector(ctx, dim):
    P = _P()
    m, beta = 8, 2.0  # small m: the rounding-level w_1 stays far below the 1e-14 breakdown threshold
    f2, lam2 = _eigvec_2d(m, beta)
    if dim == 2:
        f, lam = f2, lam2
    else:  # u x u x u, eigenvalue 3 lambda_1
        a, b, c = O.stencil_coeffs(m, beta)
        i = np.arange(1, m + 1)
        u = (b / c) ** (i / 2.0) * np.sin(i * np.pi / (m + 1))
        f = np.einsum("i,j,k->ijk", u, u, u).ravel()
        f /= np.linalg.norm(f)
        lam = 3.0 * (a - 2.0 * np.sqrt(b * c) * np.cos(np.pi / (m + 1)))
    Ao = O.stencil_matrix(dim, m, beta)
    assert np.linalg.norm(Ao @ f - lam * f) <= 1e-13 * lam           # the closed form is an eigenpair
    res = ctx.sgmres_solve(P.StencilOperator(dim, m, beta), f, d=10, k=2, s=20, seed=1, tol=1e-8, max_cycles=2)
    orc = O.sgmres_solve(lambda v: Ao @ v, f, 10, 2, 20, 8, 1, tol=1e-8, max_cycles=2)
    assert res.info["flags"] & _P()._lib.SKS_WARN_BREAKDOWN and orc["flags"] & 2
    assert res.converged and res.info["columns"] == orc["columns"] == 1
    np.testing.assert_allclose(res.x, f / lam, rtol=0, atol=1e-12 * np.abs(f / lam).max())
    np.testing.assert_allclose(res.x, orc["x"], rtol=0, atol=1e-12 * np.abs(orc["x"]).max())


def test_srr_invariant_start_vector_is_rejected(ctx):
    P = _P()
    f, _ = _eigvec_2d(8, 2.0)
    with pytest.raises(P.SksError) as e:
        ctx.srr_eigs(P.StencilOperator(2, 8, 2.0), f, d=20, k=2, s=40, nev=4)
    assert e.value.status == -1


def test_sgmres_single_column(ctx):
    P = _P()
    m, beta = 16, 5.0
    f = rhs_normal(m * m, 3)
    Ao = O.stencil_matrix(2, m, beta)
    res = ctx.sgmres_solve(P.StencilOperator(2, m, beta), f, d=1, k=1, s=4, zeta=4, seed=3, tol=1e-8,
                           max_cycles=4)
    orc = O.sgmres_solve(lambda v: Ao @ v, f, 1, 1, 4, 4, 3, tol=1e-8, max_cycles=4)
    assert res.info["cycles"] == orc["cycles"] == 4
    np.testing.assert_allclose(res.hist_true, orc["hist_true"], rtol=1e-10)
    np.testing.assert_allclose(res.x, orc["x"], rtol=0, atol=1e-10 * np.abs(orc["x"]).max())


@pytest.mark.parametrize("dim,m", [(2, 20), (3, 10)])
def test_full_orthogonalisation_k_ge_d(ctx, dim, m):
    """k = 8 >= d = 8: the truncated recurrence is full Arnoldi, so the basis is orthonormal
    (oracle pin: ||B^T B - I|| < 1e-12) and equals the oracle's column by column."""
    P = _P()
    r0 = rhs_normal(m ** dim, 5)
    Ao = O.stencil_matrix(dim, m, 3.0)
    B, H = ctx.basis(P.StencilOperator(dim, m, 3.0), r0, k=8, ncols=8)
    assert np.abs(B.T @ B - np.eye(8)).max() <= 1e-12
    ref = O.partial_arnoldi(lambda v: Ao @ v, r0, 8, 8)
    assert np.abs(B - ref["B"]).max() <= 1e-10 * np.abs(ref["B"]).max()


def test_smallest_stencil_m2(ctx):
    """m = 2 (n = 4 in 2D, 8 in 3D): every point touches the Dirichlet boundary; d = n-1 columns."""
    P = _P()
    for dim in (2, 3):
        n = 2 ** dim
        f = rhs_normal(n, 7)
        Ao = O.stencil_matrix(dim, 2, 1.0)
        res = ctx.sgmres_solve(P.StencilOperator(dim, 2, 1.0), f, d=n - 1, k=2, s=2 * n, seed=7, tol=1e-12,
                               max_cycles=6)
        orc = O.sgmres_solve(lambda v: Ao @ v, f, n - 1, 2, 2 * n, 8, 7, tol=1e-12, max_cycles=6)
        x_exact = np.linalg.solve(Ao.toarray(), f)
        assert res.info["cycles"] == orc["cycles"]
        np.testing.assert_allclose(res.x, orc["x"], rtol=0, atol=1e-9 * np.abs(x_exact).max())
        assert np.linalg.norm(res.x - x_exact) <= 1e-9 * np.linalg.norm(x_exact)


def test_srr_rejects_unknown_stabilize_mode(ctx):
    """opts.stabilize outside SKS_SRR_STABILIZE_* is an argument error (sks.h), checked in the C ABI."""
    import ctypes as C
    P = _P()
    L = P._lib
    A = P.StencilOperator(2, 16, 5.0)
    op, keep = A.struct()
    v0 = np.ascontiguousarray(start_vector(256, 4))
    opts = L.SrrOpts(20, 2, 40, 8, 4, 1e14, 0, 0, 7, 0, 0.0, 0.0, 0.0)
    out = [np.zeros(5) for _ in range(4)]
    info = L.SrrInfo()
    st = ctx.lib.sks_srr_eigs(ctx.h, C.byref(op), v0.ctypes.data, C.byref(opts), 4, 5, out[0].ctypes.data,
                              out[1].ctypes.data, out[2].ctypes.data, out[3].ctypes.data, None, None, C.byref(info))
    assert st == -1


def test_srr_stabilized_rank_below_two_is_rejected(ctx):
    """cond_tol = 1 keeps only sigma_1 (rank 1): no 2-column Rayleigh-Ritz problem -> SKS_EINVAL."""
    P = _P()
    with pytest.raises(P.SksError) as e:
        ctx.srr_eigs(P.StencilOperator(2, 16, 5.0), start_vector(256, 4), d=20, k=2, s=40, nev=4, seed=4,
                     cond_tol=1.0, stabilize="always")
    assert e.value.status == -1


def test_srr_stabilized_rank_below_nev(ctx):
    """Truncation to rank 3 < nev = 4 (tol placed between sigma_1/sigma_3 and sigma_1/sigma_4 of the
    oracle's SB): at most rank (+ a conjugate partner) pairs come back, equal to the oracle's rank-3
    pencil (QZ)."""
    P = _P()
    m, beta, d = 16, 5.0, 20
    v0 = start_vector(m * m, 4)
    A = O.stencil_matrix(2, m, beta)
    ref = O.srr_eigs(lambda v: A @ v, v0, d, 2, 2 * d, 8, 4, 4, stabilize="always", tol=1e14)
    sig = ref["sigma"]
    tol = np.sqrt((sig[0] / sig[2]) * (sig[0] / sig[3]))
    orc = O.srr_eigs(lambda v: A @ v, v0, d, 2, 2 * d, 8, 4, 4, stabilize="always", tol=tol)
    assert orc["rank"] == 3
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=2, s=2 * d, nev=4, seed=4, cond_tol=tol,
                       stabilize="always")
    assert out["info"]["rank"] == 3 and 1 <= out["info"]["nev_out"] <= 4
    err = max(np.abs(orc["theta_all"] - t).min() / np.abs(t) for t in out["theta"])
    assert err <= 1e-8


# ---------------------------------------------------------------- round-2 features: edge cases
def test_block_srr_depth_one_and_block_one(ctx):
    """p = 1 (d = b: the basis is Omega itself, S A B from the extra block B_2) and b = 1 (the single-vector
    Chebyshev recurrence without normalisation) both equal the oracle's block sRR."""
    import paper_2111_00113_b200 as P
    from inputs import start_block
    m, beta = 48, 10.0
    A = O.stencil_matrix(2, m, beta)
    box = O.spectral_box(2, m, beta)
    for b, p in ((12, 1), (1, 14)):
        Om = start_block(m * m, b, 8)
        out = ctx.srr_eigs(P.StencilOperator(2, m, beta), Om, d=b * p, k=2, s=2 * b * p, nev=4, zeta=8, seed=1,
                           basis="block_chebyshev")
        ref = O.srr_eigs_block(lambda v: A @ v, Om, p, *box, 2 * b * p, 8, 1, 4)
        assert len(out["theta"]) == len(ref["theta"])
        assert (np.abs(out["theta"] - ref["theta"]) / np.abs(ref["theta"])).max() <= 1e-8, (b, p)


def test_whiten_never_triggered_equals_plain(ctx):
    """cond_tol far above every kappa_2(T_j): whitening never fires and the run is the plain one, bit for bit."""
    import paper_2111_00113_b200 as P
    f = rhs_normal(1024, 0)
    A = P.StencilOperator(2, 32, 20.0)
    kw = dict(d=40, k=2, s=80, zeta=8, seed=0, tol=1e-12, max_cycles=1, early_exit_factor=0.0, cond_tol=1e12)
    w = ctx.sgmres_solve(A, f, whiten=True, **kw)
    p = ctx.sgmres_solve(A, f, **kw)
    assert not (w.info["flags"] & P._lib.SKS_INFO_WHITEN)
    assert np.array_equal(np.asarray(w.x), np.asarray(p.x))


def test_whiten_threshold_below_first_columns_stops_cleanly(ctx):
    """A threshold crossed at once (kappa_2(T_2) > tol): whitening keeps J = 1 column, regenerates, crosses again
    at the same J and ends the cycle (reading O36) -- a valid, finite solution from one column."""
    import paper_2111_00113_b200 as P
    f = rhs_normal(1024, 0)
    Ao = O.stencil_matrix(2, 32, 20.0)
    res = ctx.sgmres_solve(P.StencilOperator(2, 32, 20.0), f, d=40, k=2, s=80, zeta=8, seed=0, tol=1e-12,
                           max_cycles=1, early_exit_factor=0.0, cond_tol=1.0 + 1e-9, whiten=True)
    assert 1 <= res.info["columns"] <= 40
    rel = np.linalg.norm(f - Ao @ np.asarray(res.x)) / np.linalg.norm(f)
    assert np.isfinite(rel) and rel <= 1.0


@pytest.mark.parametrize("n,c,s", [(1009, 3, 50), (4096, 32, 64), (97, 1, 97)])
def test_srft_apply_prime_and_full_batches(ctx, n, c, s):
    """The pruned DFT's degenerate factorisations: prime n (n1 = 1: stage 2 is the direct DFT), a full 32-column
    batch, and s = n (every DCT coordinate sampled: an orthogonal transform, ||S x|| = ||x||)."""
    M = np.random.default_rng(n).standard_normal((n, c))
    SM = ctx.srft_apply(M, s=s, seed=2, cycle=0)
    ref = O.srft_apply(M, s, 2, 0)
    assert np.linalg.norm(SM - ref) / np.linalg.norm(ref) <= 1e-12
    if s == n:
        np.testing.assert_allclose(np.linalg.norm(SM, axis=0), np.linalg.norm(M, axis=0), rtol=1e-12)


def test_loopback_group_limits():
    import paper_2111_00113_b200 as P
    with pytest.raises(P.SksError):
        P.LoopbackGroup(17)
    g = P.LoopbackGroup(1)             # a one-rank group behaves like a plain context
    c = P.Context(0, 0, loopback=g)
    f = rhs_normal(1024, 0)
    r = c.sgmres_solve(P.StencilOperator(2, 32, 20.0), f, d=20, k=2, s=40, zeta=8, seed=0, max_cycles=1)
    assert np.isfinite(r.info["rel_res_true"])
    c.close()
    g.close()
