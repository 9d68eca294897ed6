"""GPU <-> oracle parity through the C-ABI (run on a B200 under gpurun: -m gpu).

Tolerances (BASELINE.json north_star):
  * S M for a given M: relative Frobenius error <= 1e-12;  S tables bit-exact (integer work);
  * first 20 basis columns: <= 1e-10 relative;
  * final relative residual ||Ax - f||/||f|| recomputed by the ORACLE's operator: <= 1e-8
    (configs that restart to tol) and within 2x of the oracle's own final residual;
  * Ritz values: <= 1e-8 relative (matched canonically, reading O23).
Sizes span several tiles and ragged tails; the full-size configs are checked on
properties that hold at any size (true residual via the oracle's SpMV).
"""
import numpy as np
import pytest

import oracle as O
from inputs import get_config, rhs_normal, start_vector, random_csr_c4

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


# ---------------------------------------------------------------- sketch
@pytest.mark.parametrize("s,zeta,seed,cycle,rb", [(600, 8, 2, 0, 0), (120, 8, 0, 3, 12345), (400, 8, 1, 13, 7),
                                                  (40, 3, 9, 0, 0), (17, 16, 5, 1, 99), (2048, 8, 4, 2, 3)])
def test_sketch_table_bit_exact(ctx, s, zeta, seed, cycle, rb):
    count = 5000
    q, sg = ctx.sketch_table(rb, count, s=s, zeta=zeta, seed=seed, cycle=cycle)
    qo, so = O.sketch_table(np.arange(rb, rb + count), s, zeta, seed, cycle)
    assert np.array_equal(q, qo)
    assert np.array_equal(sg.astype(np.float64), so)


@pytest.mark.parametrize("n,c,s,rb", [(1024, 1, 120, 0), (50_001, 40, 600, 0), (99_999, 32, 400, 4096 * 7),
                                      (777, 5, 600, 3), (300_000, 7, 2048, 0),
                                      # narrow batches (half- / quarter-warp gathers): J = 13, 16, 44 = 32 + 12, 3
                                      (60_001, 13, 600, 0), (40_000, 16, 400, 100), (70_003, 44, 600, 9), (513, 3, 600, 0)])
def test_sketch_apply_parity(ctx, n, c, s, rb):
    rng = np.random.default_rng(n + c)
    M = rng.standard_normal((n, c))
    SM = ctx.sketch_apply(M, s=s, zeta=8, seed=2, cycle=1, row_begin=rb, n_global=rb + n)
    ref = O.sketch_apply(M, s, 8, 2, 1, row_begin=rb, n=rb + n)
    err = np.linalg.norm(SM - ref) / np.linalg.norm(ref)
    assert err <= 1e-12, err


def test_sketch_apply_device_tensor_and_determinism(ctx):
    import torch
    rng = np.random.default_rng(0)
    M = rng.standard_normal((70_000, 33))
    Mt = torch.from_numpy(M).cuda()
    a = ctx.sketch_apply(Mt, s=300, zeta=8, seed=3).cpu().numpy()
    b = ctx.sketch_apply(Mt, s=300, zeta=8, seed=3).cpu().numpy()
    assert np.array_equal(a, b)            # bitwise reproducible (fixed-order reductions)
    ref = O.sketch_apply(M, 300, 8, 3)
    assert np.linalg.norm(a - ref) / np.linalg.norm(ref) <= 1e-12


# ---------------------------------------------------------------- operator
@pytest.mark.parametrize("dim,m,beta", [(2, 32, 20.0), (2, 77, 50.0), (3, 20, 30.0), (3, 9, 3.0)])
def test_apply_stencil(ctx, dim, m, beta):
    P = _P()
    x = np.random.default_rng(1).standard_normal(m ** dim)
    y = ctx.apply_operator(P.StencilOperator(dim, m, beta), x)
    ref = O.stencil_matrix(dim, m, beta) @ x
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)


def test_apply_csr(ctx):
    P = _P()
    n = 20_000
    rp, ci, v, f = random_csr_c4(n, seed=3)
    y = ctx.apply_operator(P.CsrOperator(rp, ci, v, n), f)
    ref = O.csr_matrix(rp, ci, v, n) @ f
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)


# ---------------------------------------------------------------- basis (first 20 columns <= 1e-10)
@pytest.mark.parametrize("case", ["C1", "C2s", "C3s", "C4s", "k1", "k8", "3d_even", "3d_k4", "3d_k8", "3d_tiny"])
def test_basis_first_columns(ctx, case):
    """Odd m runs the generic stencil kernels; even m the TMA kernels (3D: z-march, ragged
    32 x 16 tiles in x/y and plane ranges split across CTAs; k = 4, 8 use 2 and 1 planes/step)."""
    P = _P()
    if case == "3d_even":
        A, Ao, k, n = P.StencilOperator(3, 50, 30.0), O.stencil_matrix(3, 50, 30.0), 2, 50 ** 3
    elif case == "3d_k4":
        A, Ao, k, n = P.StencilOperator(3, 36, 20.0), O.stencil_matrix(3, 36, 20.0), 4, 36 ** 3
    elif case == "3d_k8":
        A, Ao, k, n = P.StencilOperator(3, 28, 10.0), O.stencil_matrix(3, 28, 10.0), 8, 28 ** 3
    elif case == "3d_tiny":
        A, Ao, k, n = P.StencilOperator(3, 6, 3.0), O.stencil_matrix(3, 6, 3.0), 2, 6 ** 3
    elif case == "C1":
        A, Ao, k, n = P.StencilOperator(2, 32, 20.0), O.stencil_matrix(2, 32, 20.0), 2, 1024
    elif case == "C2s":
        A, Ao, k, n = P.StencilOperator(2, 130, 50.0), O.stencil_matrix(2, 130, 50.0), 4, 130 ** 2
    elif case == "C3s":
        A, Ao, k, n = P.StencilOperator(3, 37, 30.0), O.stencil_matrix(3, 37, 30.0), 2, 37 ** 3
    elif case == "C4s":
        n = 30_000
        rp, ci, v, _ = random_csr_c4(n, seed=3)
        A, Ao, k = P.CsrOperator(rp, ci, v, n), O.csr_matrix(rp, ci, v, n), 2
    elif case == "k1":
        A, Ao, k, n = P.StencilOperator(2, 50, 10.0), O.stencil_matrix(2, 50, 10.0), 1, 2500
    else:
        A, Ao, k, n = P.StencilOperator(2, 40, 5.0), O.stencil_matrix(2, 40, 5.0), 8, 1600
    r0 = rhs_normal(n, 7)
    B, H = ctx.basis(A, r0, k=k, ncols=20)
    ref = O.partial_arnoldi(lambda v: Ao @ v, r0, 20, k)
    err = np.abs(B - ref["B"]).max() / np.abs(ref["B"]).max()
    assert err <= 1e-10, err
    Ho = ref["H"][:20, :19]
    assert np.abs(H - Ho).max() <= 1e-10 * np.abs(Ho).max()


# ---------------------------------------------------------------- sGMRES
def test_sgmres_c1_parity(ctx):
    P = _P()
    c = get_config("C1")
    f = rhs_normal(c.n, c.seed)
    A = O.stencil_matrix(2, c.m, c.beta)
    res = ctx.sgmres_solve(P.StencilOperator(2, c.m, c.beta), f, d=c.d, k=c.k, s=c.s, zeta=c.zeta, seed=c.seed,
                           tol=c.tol, max_cycles=c.max_cycles)
    orc = O.sgmres_solve(lambda v: A @ v, f, c.d, c.k, c.s, c.zeta, c.seed, tol=c.tol, max_cycles=c.max_cycles)
    rel_gpu = np.linalg.norm(f - A @ res.x) / np.linalg.norm(f)      # recomputed by the oracle
    assert rel_gpu <= 2 * orc["rel_res_true"] and orc["rel_res_true"] <= 2 * rel_gpu
    assert abs(res.info["rel_res_true"] - rel_gpu) <= 1e-6 * rel_gpu
    assert res.info["columns"] == orc["columns"]
    np.testing.assert_allclose(res.hist, orc["hist_est"], rtol=1e-6)
    np.testing.assert_allclose(res.x, orc["x"], rtol=0, atol=1e-6 * np.abs(orc["x"]).max())


def test_sgmres_c1_restarted_to_tol(ctx):
    P = _P()
    c = get_config("C1")
    f = rhs_normal(c.n, c.seed)
    A = O.stencil_matrix(2, c.m, c.beta)
    res = ctx.sgmres_solve(P.StencilOperator(2, c.m, c.beta), f, d=c.d, k=c.k, s=c.s, seed=c.seed, tol=1e-8,
                           max_cycles=5)
    orc = O.sgmres_solve(lambda v: A @ v, f, c.d, c.k, c.s, c.zeta, c.seed, tol=1e-8, max_cycles=5)
    rel_gpu = np.linalg.norm(f - A @ res.x) / np.linalg.norm(f)
    assert res.converged and rel_gpu <= 1e-8
    assert rel_gpu <= 2 * orc["rel_res_true"] and orc["rel_res_true"] <= 2 * rel_gpu
    assert res.info["cycles"] == orc["cycles"] and res.info["columns"] == orc["columns"]
    np.testing.assert_allclose(res.hist_true, orc["hist_true"], rtol=1e-4)


def test_sgmres_csr_small(ctx):
    P = _P()
    n = 40_000
    rp, ci, v, f = random_csr_c4(n, seed=3)
    Ao = O.csr_matrix(rp, ci, v, n)
    res = ctx.sgmres_solve(P.CsrOperator(rp, ci, v, n), f, d=40, k=2, s=80, seed=3, tol=1e-8, max_cycles=3)
    orc = O.sgmres_solve(lambda x: Ao @ x, f, 40, 2, 80, 8, 3, tol=1e-8, max_cycles=3)
    rel_gpu = np.linalg.norm(f - Ao @ res.x) / np.linalg.norm(f)
    assert rel_gpu <= 1e-8 and rel_gpu <= 2 * orc["rel_res_true"] and orc["rel_res_true"] <= 2 * rel_gpu
    assert res.info["columns"] == orc["columns"]


def test_sgmres_3d_small_restarts(ctx):
    P = _P()
    m = 24
    f = rhs_normal(m ** 3, 2)
    Ao = O.stencil_matrix(3, m, 30.0)
    res = ctx.sgmres_solve(P.StencilOperator(3, m, 30.0), f, d=60, k=2, s=120, seed=2, tol=1e-8, max_cycles=10)
    orc = O.sgmres_solve(lambda x: Ao @ x, f, 60, 2, 120, 8, 2, tol=1e-8, max_cycles=10)
    rel_gpu = np.linalg.norm(f - Ao @ res.x) / np.linalg.norm(f)
    assert res.converged and rel_gpu <= 1e-8
    assert rel_gpu <= 2 * orc["rel_res_true"] and orc["rel_res_true"] <= 2 * rel_gpu
    assert res.info["cycles"] == orc["cycles"]


def test_sgmres_host_and_device_buffers_agree(ctx):
    import torch
    P = _P()
    c = get_config("C1")
    f = rhs_normal(c.n, c.seed)
    A = P.StencilOperator(2, c.m, c.beta)
    r1 = ctx.sgmres_solve(A, f, d=c.d, k=c.k, s=c.s, seed=c.seed, max_cycles=1)
    r2 = ctx.sgmres_solve(A, torch.from_numpy(f).cuda(), d=c.d, k=c.k, s=c.s, seed=c.seed, max_cycles=1)
    assert np.array_equal(r1.x, r2.x.cpu().numpy())   # deterministic, same kernels


# ---------------------------------------------------------------- sRR
def _match(th_gpu, th_orc):
    err = 0.0
    for t in th_gpu:
        j = np.argmin(np.abs(th_orc - t))
        err = max(err, abs(th_orc[j] - t) / abs(th_orc[j]))
    return err


@pytest.mark.parametrize("m,beta,d", [(32, 10.0, 40), (64, 10.0, 80)])
def test_srr_parity_small(ctx, m, beta, d):
    P = _P()
    n = m * m
    v0 = start_vector(n, 4)
    Ao = O.stencil_matrix(2, m, beta)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=2, s=2 * d, nev=10, seed=4)
    orc = O.srr_eigs(lambda x: Ao @ x, v0, d, 2, 2 * d, 8, 4, 10)
    assert _match(out["theta"], orc["theta_all"]) <= 1e-8
    # same selection (canonical order, O23)
    assert len(out["theta"]) == len(orc["theta"])
    np.testing.assert_allclose(np.sort_complex(out["theta"]), np.sort_complex(orc["theta"]), rtol=1e-8)
    np.testing.assert_allclose(np.sort(out["res_true"]), np.sort(orc["res_true"]), rtol=1e-4)
    np.testing.assert_allclose(np.sort(out["res_est"]), np.sort(orc["res_est"]), rtol=1e-4)


def test_srr_closed_form_full_dimension(ctx):
    """d = n with k >= d-1 (full orthogonalisation) on a 2D grid.  The 2D spectrum
    mu_p + mu_q (BASELINE north_star closed form) has repeated values, so the Krylov space
    of one vector has dimension = number of DISTINCT eigenvalues: the basis breaks down
    there (reading O10) and every Ritz value is one of the distinct eigenvalues."""
    P = _P()
    m, beta = 3, 3.0
    n = m * m
    v0 = start_vector(n, 4)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=n, k=8, s=2 * n, nev=9, seed=4)
    ev = O.closed_form_eigs(2, m, beta)
    distinct = np.unique(np.round(ev / ev.max(), 12)) * ev.max()
    assert out["info"]["flags"] & 2              # SKS_WARN_BREAKDOWN
    assert out["info"]["columns"] == distinct.size
    assert np.abs(out["theta"].imag).max() <= 1e-9 * ev.max()
    np.testing.assert_allclose(np.sort(out["theta"].real), distinct, rtol=1e-9)


# ---------------------------------------------------------------- Chebyshev basis (NEXT(1))
@pytest.mark.parametrize("dim,m,beta,d", [(2, 32, 20.0, 60), (2, 33, 20.0, 60), (3, 24, 30.0, 60), (3, 19, 10.0, 40)])
def test_sgmres_chebyshev_parity(ctx, dim, m, beta, d):
    """Eq. Chebrecurse with the closed-form spectral box: same restarts, history
    and solution as the oracle's Chebyshev sGMRES (even m: TMA kernels, odd m: generic)."""
    P = _P()
    n = m ** dim
    f = rhs_normal(n, 2)
    Ao = O.stencil_matrix(dim, m, beta)
    box = O.spectral_box(dim, m, beta)
    res = ctx.sgmres_solve(P.StencilOperator(dim, m, beta), f, d=d, k=2, s=2 * d, seed=2, tol=1e-8, max_cycles=8,
                           basis="chebyshev")
    orc = O.sgmres_solve(lambda x: Ao @ x, f, d, 2, 2 * d, 8, 2, tol=1e-8, max_cycles=8, cheb=box)
    rel_gpu = np.linalg.norm(f - Ao @ res.x) / np.linalg.norm(f)
    assert rel_gpu <= 2 * orc["rel_res_true"] and orc["rel_res_true"] <= 2 * rel_gpu
    assert res.info["cycles"] == orc["cycles"] and res.info["columns"] == orc["columns"]
    np.testing.assert_allclose(res.hist, orc["hist_est"], rtol=1e-6)


def test_srr_chebyshev_parity(ctx):
    P = _P()
    m, beta, d = 48, 10.0, 60
    v0 = start_vector(m * m, 4)
    Ao = O.stencil_matrix(2, m, beta)
    box = O.spectral_box(2, m, beta)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=2, s=2 * d, nev=6, seed=4, basis="chebyshev")
    bas = O.chebyshev_basis(lambda x: Ao @ x, v0, d, *box)
    orc = O.srr_from_basis(lambda x: Ao @ x, bas["B"], bas["M"], O.sketch_matrix(m * m, 2 * d, 8, 4, 0), 6)
    assert _match(out["theta"], orc["theta_all"]) <= 1e-8
    np.testing.assert_allclose(np.sort(out["res_true"]), np.sort(orc["res_true"]), rtol=1e-4)


# ---------------------------------------------------------------- adaptive restarting (NEXT(2))
def test_sgmres_adaptive_restart_parity(ctx):
    """Adaptive restarting (reading O31): the first cycle ends at the same column as the
    oracle's exact rule -- cond_tol is put at the geometric midpoint of two consecutive kappa_2(T_j)
    (2.3x apart with a k = 1 basis), so the device's power-iteration estimate cannot straddle it --
    with the same solution; restarted to 1e-8 it converges (true residual by the oracle's operator)."""
    from scipy.linalg import svdvals
    P = _P()
    m, beta, d, k, s = 32, 20.0, 40, 1, 80
    A = O.stencil_matrix(2, m, beta)
    f = rhs_normal(m * m, 0)
    out = O.sgmres_cycle(lambda v: A @ v, f, np.zeros_like(f), d, k, s, 8, 0, 0, early_exit_factor=0.0)
    kap = [svdvals(out["C"][:, :j]) for j in (20, 21)]
    tol_k = float(np.sqrt((kap[0][0] / kap[0][-1]) * (kap[1][0] / kap[1][-1])))
    Ag = P.StencilOperator(2, m, beta)
    res = ctx.sgmres_solve(Ag, f, d=d, k=k, s=s, seed=0, tol=1e-8, max_cycles=1, cond_tol=tol_k,
                           adaptive_restart=True, early_exit_factor=0.0)
    orc = O.sgmres_solve(lambda v: A @ v, f, d, k, s, 8, 0, tol=1e-8, max_cycles=1, cond_tol=tol_k,
                         adaptive=True, early_exit_factor=0.0)
    assert res.info["columns"] == orc["columns"] == 20
    assert res.info["flags"] & P._lib.SKS_INFO_ADAPTIVE_RESTART and orc["flags"] & O.INFO_ADAPTIVE
    np.testing.assert_allclose(res.x, orc["x"], rtol=0, atol=1e-8 * np.abs(orc["x"]).max())
    full = ctx.sgmres_solve(Ag, f, d=d, k=k, s=s, seed=0, tol=1e-8, max_cycles=80, cond_tol=tol_k,
                            adaptive_restart=True)
    rel = np.linalg.norm(f - A @ full.x) / np.linalg.norm(f)
    assert full.converged and rel <= 1e-8


# ---------------------------------------------------------------- SRFT sketch (NEXT(4), reading O32)
@pytest.mark.parametrize("n,c,s", [(1024, 1, 120), (777, 5, 40), (50_001, 33, 400), (262_144, 3, 600)])
def test_srft_apply_parity(ctx, n, c, s):
    rng = np.random.default_rng(n + c)
    M = rng.standard_normal((n, c))
    SM = ctx.srft_apply(M, s=s, seed=3, cycle=2)
    ref = O.srft_apply(M, s, 3, 2)
    assert np.linalg.norm(SM - ref) / np.linalg.norm(ref) <= 1e-12


def test_sgmres_srft_parity(ctx):
    P = _P()
    c = get_config("C1")
    f = rhs_normal(c.n, c.seed)
    A = O.stencil_matrix(2, c.m, c.beta)
    res = ctx.sgmres_solve(P.StencilOperator(2, c.m, c.beta), f, d=c.d, k=c.k, s=c.s, seed=c.seed, tol=1e-8,
                           max_cycles=6, sketch="srft")
    orc = O.sgmres_solve(lambda v: A @ v, f, c.d, c.k, c.s, c.zeta, c.seed, tol=1e-8, max_cycles=6, sketch="srft")
    rel = np.linalg.norm(f - A @ res.x) / np.linalg.norm(f)
    assert res.converged and rel <= 1e-8
    assert res.info["cycles"] == orc["cycles"] and res.info["columns"] == orc["columns"]
    np.testing.assert_allclose(res.hist, orc["hist_est"], rtol=1e-6)


def test_srr_srft_parity(ctx):
    P = _P()
    m, beta, d = 40, 5.0, 40
    v0 = start_vector(m * m, 4)
    A = O.stencil_matrix(2, m, beta)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=2, s=2 * d, nev=6, seed=4, sketch="srft")
    orc = O.srr_eigs(lambda v: A @ v, v0, d, 2, 2 * d, 8, 4, 6, sketch="srft")
    assert _match(out["theta"], orc["theta_all"]) <= 1e-8


# ---------------------------------------------------------------- stabilised sRR (NEXT(2), reading O33)
def test_srr_stabilized_without_truncation(ctx):
    """stabilize="always" on a well-conditioned basis (kappa(T) ~ 1e1 << tol = 1e14): rank r = d, and
    the pencil Sigma^-1 U^T SAB V is similar to Mhat, so the Ritz values equal the unstabilised
    device run's and the oracle's (QZ) ones."""
    P = _P()
    m, beta, d = 32, 10.0, 40
    v0 = start_vector(m * m, 4)
    A = O.stencil_matrix(2, m, beta)
    op = P.StencilOperator(2, m, beta)
    plain = ctx.srr_eigs(op, v0, d=d, k=2, s=2 * d, nev=8, seed=4)
    out = ctx.srr_eigs(op, v0, d=d, k=2, s=2 * d, nev=8, seed=4, stabilize="always")
    orc = O.srr_eigs(lambda v: A @ v, v0, d, 2, 2 * d, 8, 4, 8, stabilize="always", tol=1e14)
    assert out["info"]["flags"] & P._lib.SKS_INFO_STABILIZED and not plain["info"]["flags"] & P._lib.SKS_INFO_STABILIZED
    assert out["info"]["rank"] == d == orc["rank"] and plain["info"]["rank"] == d
    assert _match(out["theta"], plain["theta"]) <= 1e-10
    assert _match(out["theta"], orc["theta_all"]) <= 1e-8
    np.testing.assert_allclose(np.sort(out["res_true"]), np.sort(orc["res_true"]), rtol=1e-4)
    np.testing.assert_allclose(np.sort(out["res_est"]), np.sort(orc["res_est"]), rtol=1e-4)


@pytest.mark.parametrize("mode", ["always", "if_ill"])
def test_srr_stabilized_ill_conditioned_basis(ctx, mode):
    """k = 1 basis with kappa_2(T) ~ 1e17: truncation at tol = 1e8 keeps the same rank
    as the oracle's SVD (its kept / dropped singular values sit a factor >= 1.2 from the threshold,
    far above the rounding-level differences of the two bases), and the dominant Ritz values agree
    to 1e-6: the truncated subspace moves by ~u sigma_1 / (sigma_r - sigma_r+1) ~ 1e-8 between the
    two runs, times the Ritz values' condition numbers."""
    P = _P()
    m, beta, d, k, s, tol = 24, 10.0, 200, 1, 420, 1e8
    v0 = start_vector(m * m, 4)
    A = O.stencil_matrix(2, m, beta)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=k, s=s, nev=2, seed=4, cond_tol=tol,
                       stabilize=mode)
    orc = O.srr_eigs(lambda v: A @ v, v0, d, k, s, 8, 4, 2, stabilize="always", tol=tol)
    assert out["info"]["flags"] & P._lib.SKS_INFO_STABILIZED
    assert out["info"]["rank"] == orc["rank"] < d
    np.testing.assert_allclose(out["theta"], orc["theta"], rtol=1e-6)
    ev = np.linalg.eigvals(A.toarray())
    lam1 = ev[np.argmax(np.abs(ev))]
    assert abs(out["theta"][0] - lam1) <= 1e-5 * abs(lam1)
    assert out["res_true"][0] <= 1e-5 * abs(lam1)


def test_srr_stabilize_if_ill_leaves_well_conditioned_runs_alone(ctx):
    P = _P()
    m, beta, d = 32, 10.0, 40
    v0 = start_vector(m * m, 4)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=2, s=2 * d, nev=4, seed=4, stabilize="if_ill")
    assert not out["info"]["flags"] & P._lib.SKS_INFO_STABILIZED and out["info"]["rank"] == d
