"""GPU checks at the FULL BASELINE sizes, in the launch configuration bench.py times (the
library's default grids and streams), against what the oracle can compute at that size:

  * the true relative residual of the GPU solution, recomputed with the ORACLE's operator
    (scipy sparse matvec), for C2 (13-14 restart cycles), C3 (bench) and C4 (random CSR);
  * the first 20 basis columns of C3 and C5 against the oracle's truncated Arnoldi (20 SpMVs);
  * S M at full C3 size against the oracle's sketch (same hashed S), sampled on 3 columns;
  * the C5 sRR Ritz pairs: every reported true residual ||A x - theta x|| / ||x|| recomputed by
    the oracle's operator from the returned Ritz vectors, the canonical |theta| order (O23),
    and the top Ritz value against the closed-form largest eigenvalue (Kronecker sum).
Tolerances: BASELINE north_star (residual <= 1e-8, basis 1e-10, S M 1e-12).
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


def _op(cfg):
    import paper_2111_00113_b200 as P
    if cfg.op == "csr":
        rp, ci, v, f = random_csr_c4(cfg.n, seed=cfg.seed)
        return P.CsrOperator(rp, ci, v, cfg.n), O.csr_matrix(rp, ci, v, cfg.n), f
    dim = 3 if cfg.op == "stencil3d" else 2
    return P.StencilOperator(dim, cfg.m, cfg.beta), O.stencil_matrix(dim, cfg.m, cfg.beta), None


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
def test_full_size_true_residual(ctx, name):
    import torch
    cfg = get_config(name)
    A, Ao, f = _op(cfg)
    if f is None:
        f = rhs_normal(cfg.n, cfg.seed)
    res = ctx.sgmres_solve(A, torch.from_numpy(f).cuda(), d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta,
                           seed=cfg.seed, tol=cfg.tol, max_cycles=cfg.max_cycles)
    x = res.x.cpu().numpy()
    rel = np.linalg.norm(f - Ao @ x) / np.linalg.norm(f)     # oracle operator
    assert res.converged and rel <= cfg.tol, (rel, res.info)
    assert abs(res.info["rel_res_true"] - rel) <= 1e-3 * rel
    # per-cycle true residuals are decreasing and the last one is the reported value
    ht = res.hist_true
    assert len(ht) == res.info["cycles"] and abs(ht[-1] - res.info["rel_res_true"]) <= 1e-12 * ht[-1]


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_full_size_first_basis_columns(ctx, name):
    cfg = get_config(name)
    A, Ao, _ = _op(cfg)
    r0 = rhs_normal(cfg.n, cfg.seed) if cfg.method == "sgmres" else start_vector(cfg.n, cfg.seed)
    B, H = ctx.basis(A, r0, k=cfg.k, ncols=20)
    ref = O.partial_arnoldi(lambda v: Ao @ v, r0, 20, cfg.k)
    err = np.abs(B - ref["B"]).max() / np.abs(ref["B"]).max()
    assert err <= 1e-10, err
    Ho = ref["H"][:20, :19]
    assert np.abs(H - Ho).max() <= 1e-10 * np.abs(Ho).max()


def test_full_size_sketch_sampled(ctx):
    cfg = get_config("C3")
    rng = np.random.default_rng(5)
    M = rng.standard_normal((cfg.n, 3))
    SM = ctx.sketch_apply(M, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, cycle=1)
    ref = O.sketch_apply(M, cfg.s, cfg.zeta, cfg.seed, 1)
    assert np.linalg.norm(SM - ref) / np.linalg.norm(ref) <= 1e-12


def test_full_size_srr_ritz_residuals(ctx):
    cfg = get_config("C5")
    A, Ao, _ = _op(cfg)
    v0 = start_vector(cfg.n, cfg.seed)
    out = ctx.srr_eigs(A, v0, d=cfg.d, k=cfg.k, s=cfg.s, nev=cfg.nev, zeta=cfg.zeta, seed=cfg.seed,
                       want_vectors=True)
    th = out["theta"]
    Xr, Xi = out["X"]
    Xr = Xr.cpu().numpy() if hasattr(Xr, "cpu") else np.asarray(Xr)
    Xi = Xi.cpu().numpy() if hasattr(Xi, "cpu") else np.asarray(Xi)
    assert len(th) >= cfg.nev
    mags = np.abs(th)
    assert np.all(np.diff(mags) <= 1e-12 * mags[0])          # |theta| descending (O23)
    for i, t in enumerate(th):
        x = Xr[i] + 1j * Xi[i]
        Ax = Ao @ x.real + 1j * (Ao @ x.imag)
        r = np.linalg.norm(Ax - t * x) / np.linalg.norm(x)     # oracle operator
        assert abs(r - out["res_true"][i]) <= 1e-6 * r + 1e-12 * abs(t), (i, r, out["res_true"][i])
    # the top Ritz value approximates the largest eigenvalue of A (closed form, Kronecker sum)
    lam_max = O.closed_form_eigs(2, cfg.m, cfg.beta).max()
    assert abs(th[0].real - lam_max) <= 1e-3 * lam_max


def test_full_size_srr_stabilized_matches_unstabilised(ctx):
    """C5 with stabilize="always" (O33): kappa(SB) ~ 27 << cond_tol, so the truncated
    SVD keeps all d columns and the pencil is similar to Mhat -- the Ritz values and residuals equal
    the unstabilised run's (the two small problems differ only by rounding: 1e-10 relative)."""
    cfg = get_config("C5")
    A, _, _ = _op(cfg)
    v0 = start_vector(cfg.n, cfg.seed)
    kw = dict(d=cfg.d, k=cfg.k, s=cfg.s, nev=cfg.nev, zeta=cfg.zeta, seed=cfg.seed)
    plain = ctx.srr_eigs(A, v0, **kw)
    stab = ctx.srr_eigs(A, v0, stabilize="always", **kw)
    assert stab["info"]["rank"] == cfg.d and stab["info"]["flags"] & 16
    assert len(stab["theta"]) == len(plain["theta"])
    np.testing.assert_allclose(stab["theta"], plain["theta"], rtol=1e-10)
    np.testing.assert_allclose(stab["res_true"], plain["res_true"], rtol=1e-6)
