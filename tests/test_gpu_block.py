"""GPU parity of block Krylov sRR (Sec. "Block Krylov subspaces" P:1867-1896, "Block Chebyshev
recurrence" P:1983-2008) against oracle.srr_eigs_block, through the C ABI (sks_srr_eigs with
SKS_BASIS_BLOCK_CHEBYSHEV).

Tolerances (BASELINE north_star): Ritz values <= 1e-8 relative; the sketched and true residual estimates at
rtol 1e-6 (they are computed from the Ritz vectors, which differ by rounding: the GPU forms S A B through the
three-term recurrence, reading O34, the oracle from the explicit products A B).  The full-size case (C5B: the
C5 operator and small side with b = 30, p = 10) compares against tests/golden/oracle_C5B.json.
"""
import json
import os

import numpy as np
import pytest

import oracle as O
from inputs import get_config, start_block

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200 import build
    build.build()
    c = P.Context(0)
    yield c
    c.close()


def _oracle(dim, m, beta, Om, p, s, seed, nev, stabilize="off"):
    A = O.stencil_matrix(dim, m, beta)
    box = O.spectral_box(dim, m, beta)
    return O.srr_eigs_block(lambda v: A @ v, Om, p, *box, s, 8, seed, nev, stabilize=stabilize)


def _compare(out, ref, rtol_res=1e-6):
    th, tho = out["theta"], ref["theta"]
    assert len(th) == len(tho), (th, tho)
    rel = np.abs(th - tho) / np.abs(tho)
    assert rel.max() <= 1e-8, (rel, th, tho)
    np.testing.assert_allclose(out["res_est"], ref["res_est"], rtol=rtol_res)
    np.testing.assert_allclose(out["res_true"], ref["res_true"], rtol=rtol_res)


@pytest.mark.parametrize("dim,m,beta,b,p,nev", [(2, 64, 10.0, 4, 6, 4), (2, 96, 30.0, 8, 5, 6),
                                                (3, 16, 5.0, 3, 5, 3), (3, 24, 20.0, 5, 4, 5)])
def test_block_srr_matches_oracle(ctx, dim, m, beta, b, p, nev):
    import paper_2111_00113_b200 as P
    n = m ** dim
    Om = start_block(n, b, 7)
    d, s = b * p, 2 * b * p
    out = ctx.srr_eigs(P.StencilOperator(dim, m, beta), Om, d=d, k=2, s=s, nev=nev, zeta=8, seed=5,
                       basis="block_chebyshev")
    ref = _oracle(dim, m, beta, Om, p, s, 5, nev)
    _compare(out, ref)
    assert out["info"]["columns"] == d


def test_block_srr_stabilized_matches_oracle(ctx):
    import paper_2111_00113_b200 as P
    m, beta, b, p = 48, 12.0, 6, 5
    Om = start_block(m * m, b, 3)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), Om, d=b * p, k=2, s=2 * b * p, nev=5, zeta=8, seed=2,
                       basis="block_chebyshev", stabilize="always")
    ref = _oracle(2, m, beta, Om, p, 2 * b * p, 2, 5, stabilize="always")
    _compare(out, ref)
    assert out["info"]["flags"] & 16


def test_block_srr_device_start_block(ctx):
    """The start block may live on the device (torch tensor): same result as from the host."""
    import torch
    import paper_2111_00113_b200 as P
    Om = start_block(64 * 64, 4, 1)
    A = P.StencilOperator(2, 64, 10.0)
    kw = dict(d=24, k=2, s=48, nev=4, zeta=8, seed=5, basis="block_chebyshev")
    h = ctx.srr_eigs(A, Om, **kw)
    dv = ctx.srr_eigs(A, torch.from_numpy(np.array(Om)).cuda(), **kw)
    assert np.array_equal(h["theta"], dv["theta"])


def test_block_srr_rejects_bad_arguments(ctx):
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200.api import SksError
    from inputs import random_csr_c4
    Om = start_block(32 * 32, 5, 1)
    with pytest.raises(SksError):   # d not a multiple of the block size
        ctx.srr_eigs(P.StencilOperator(2, 32, 5.0), Om, d=12, k=2, s=24, nev=3, basis="block_chebyshev")
    rp, ci, v, _ = random_csr_c4(1000, seed=3)
    with pytest.raises(SksError):   # CSR: no closed-form spectral box, block basis is stencil-only
        ctx.srr_eigs(P.CsrOperator(rp, ci, v, 1000), start_block(1000, 2, 1), d=8, k=2, s=16, nev=3,
                     basis="block_chebyshev")


def test_block_srr_full_size_vs_oracle_golden(ctx):
    import paper_2111_00113_b200 as P
    cfg = get_config("C5B")
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_C5B.json")) as fh:
        g = json.load(fh)
    Om = start_block(cfg.n, cfg.block, cfg.seed)
    out = ctx.srr_eigs(P.StencilOperator(2, cfg.m, cfg.beta), Om, d=cfg.d, k=2, s=cfg.s, nev=cfg.nev, zeta=cfg.zeta,
                       seed=cfg.seed, basis="block_chebyshev")
    th = out["theta"]
    tho = np.asarray(g["theta_re"]) + 1j * np.asarray(g["theta_im"])
    assert cfg.nev <= len(th) <= cfg.nev + 1
    rel = np.abs(th - tho[:len(th)]) / np.abs(tho[:len(th)])
    assert rel.max() <= 1e-8, rel
    np.testing.assert_allclose(out["res_est"], g["res_est"][:len(th)], rtol=1e-4)
    np.testing.assert_allclose(out["res_true"], g["res_true"][:len(th)], rtol=1e-4)
