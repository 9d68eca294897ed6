"""Multi-rank execution of the library's OWN communication code on one GPU (VERDICT r01 "Next round"
item 7c): P contexts in one process, one host thread per rank, joined by the loopback transport (include/sks.h
sks_loopback_*; csrc/comm.cu) -- the 1D row partition, ghost planes and halo exchange, the per-rank partial sums
pre-reduced to k+3 scalars and all-reduced, the all-reduced partial sketches, the CSR all-gather and the replicated
small side all run exactly as under NCCL, with device-to-device copies ordered by events instead.

Checks (SURVEY 8(e) "Parity across P"): each rank's rows of x -- and of the first 20 basis columns -- at P = 2 and 4
equal the P = 1 result to <= 1e-10 (only reduction order changes with P); cycle and column counts are equal; sRR
Ritz values equal to 1e-10.  Uneven slabs (m = 50 over 4 ranks: 13/13/12/12 planes, hence different step grids
per rank) cover the ADVICE r01 partial-slot finding.
"""
import threading

import numpy as np
import pytest

from inputs import partition_rows, random_csr_c4

pytestmark = pytest.mark.gpu


def _run_ranks(P, fn):
    import paper_2111_00113_b200 as PK
    grp = PK.LoopbackGroup(P)
    ctxs = [PK.Context(0, r, loopback=grp) for r in range(P)]
    out, err = [None] * P, [None] * P

    def work(r):
        try:
            out[r] = fn(ctxs[r], r)
        except Exception as e:  # pragma: no cover - reported below
            err[r] = e
    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "a rank did not finish (collective mismatch?)"
    for c in ctxs:
        c.close()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    return out


def _solve(kind, m, n, beta, f, P, kw, csr=None):
    import paper_2111_00113_b200 as PK

    def fn(ctx, r):
        lo, hi = partition_rows(kind, n, m, P, r)
        if kind == "csr":
            rp, ci, v = csr
            rpl = (rp[lo:hi + 1] - rp[lo]).astype(np.int32)
            A = PK.CsrOperator(rpl, ci[rp[lo]:rp[hi]], v[rp[lo]:rp[hi]], n, lo, hi)
        else:
            A = PK.StencilOperator(3 if kind == "stencil3d" else 2, m, beta, lo, hi)
        res = ctx.sgmres_solve(A, f[lo:hi].copy(), **kw)
        return res
    return _run_ranks(P, fn)


@pytest.mark.parametrize("kind,m,P", [("stencil3d", 48, 2), ("stencil3d", 50, 4), ("stencil2d", 256, 2),
                                      ("stencil2d", 1024, 2), ("stencil3d", 33, 3)])
def test_loopback_sgmres_matches_single_rank(kind, m, P):
    dim = 3 if kind == "stencil3d" else 2
    n = m ** dim
    f = np.random.default_rng(m).standard_normal(n)
    kw = dict(d=30, k=2, s=60, zeta=8, seed=4, tol=1e-10, max_cycles=3)
    ref = _solve(kind, m, n, 20.0, f, 1, kw)[0]
    outs = _solve(kind, m, n, 20.0, f, P, kw)
    x = np.concatenate([o.x for o in outs])
    assert all(o.info["cycles"] == ref.info["cycles"] and o.info["columns"] == ref.info["columns"] for o in outs)
    assert np.abs(x - ref.x).max() <= 1e-10 * np.abs(ref.x).max(), np.abs(x - ref.x).max() / np.abs(ref.x).max()
    for o in outs:  # the replicated small side: identical on every rank
        np.testing.assert_array_equal(o.hist, outs[0].hist)
    np.testing.assert_allclose(outs[0].hist, ref.hist, rtol=1e-8)


def test_loopback_csr_matches_single_rank():
    n = 30000
    rp, ci, v, f = random_csr_c4(n, seed=3)
    kw = dict(d=20, k=2, s=40, zeta=8, seed=3, tol=1e-10, max_cycles=3)
    ref = _solve("csr", 0, n, 0.0, f, 1, kw, csr=(rp, ci, v))[0]
    outs = _solve("csr", 0, n, 0.0, f, 2, kw, csr=(rp, ci, v))
    x = np.concatenate([o.x for o in outs])
    assert np.abs(x - ref.x).max() <= 1e-10 * np.abs(ref.x).max()
    assert outs[0].info["columns"] == ref.info["columns"]


def test_loopback_basis_columns_match_single_rank():
    import paper_2111_00113_b200 as PK
    m, P = 40, 4
    n = m ** 3
    r0 = np.random.default_rng(1).standard_normal(n)

    def fn(ctx, r):
        lo, hi = partition_rows("stencil3d", n, m, P, r)
        B, H = ctx.basis(PK.StencilOperator(3, m, 30.0, lo, hi), r0[lo:hi].copy(), k=2, ncols=20)
        return B, H

    B1, H1 = _run_ranks(1, lambda ctx, r: ctx.basis(PK.StencilOperator(3, m, 30.0), r0, k=2, ncols=20))[0]
    outs = _run_ranks(P, fn)
    B = np.concatenate([o[0] for o in outs], axis=0)
    assert np.abs(B - B1).max() <= 1e-10 * np.abs(B1).max()
    for o in outs:
        assert np.abs(o[1] - H1).max() <= 1e-10 * np.abs(H1).max()


def test_loopback_srr_matches_single_rank():
    import paper_2111_00113_b200 as PK
    m, P = 128, 2
    n = m * m
    v0 = np.random.default_rng(2).standard_normal(n)

    def fn_for(P_):
        def fn(ctx, r):
            lo, hi = partition_rows("stencil2d", n, m, P_, r)
            return ctx.srr_eigs(PK.StencilOperator(2, m, 10.0, lo, hi), v0[lo:hi].copy(), d=40, k=2, s=80, nev=6,
                                zeta=8, seed=4)
        return fn
    ref = _run_ranks(1, fn_for(1))[0]
    outs = _run_ranks(P, fn_for(P))
    for o in outs:
        rel = np.abs(o["theta"] - ref["theta"]) / np.abs(ref["theta"])
        assert rel.max() <= 1e-10, rel
        np.testing.assert_allclose(o["res_true"], ref["res_true"], rtol=1e-8)


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_chebyshev_deferred_matches_single_rank(P):
    """Chebyshev basis: per column only the halo exchange; the norms and recurrence bookkeeping of
    a batch are reduced once per batch (one all-reduce of batch x (k+3) scalars).  Same x as P = 1 to 1e-10."""
    m = 48
    n = m ** 3
    f = np.random.default_rng(9).standard_normal(n)
    kw = dict(d=40, k=2, s=80, zeta=8, seed=4, tol=1e-10, max_cycles=3, basis="chebyshev")
    ref = _solve("stencil3d", m, n, 20.0, f, 1, kw)[0]
    outs = _solve("stencil3d", m, n, 20.0, f, P, kw)
    x = np.concatenate([o.x for o in outs])
    assert all(o.info["columns"] == ref.info["columns"] for o in outs)
    assert np.abs(x - ref.x).max() <= 1e-10 * np.abs(ref.x).max()


def test_loopback_block_srr_and_stabilized_match_single_rank():
    """Block Chebyshev sRR (per-column halo exchange of every block column) and the stabilised sRR (replicated
    Jacobi SVD of the all-reduced SB) at P = 2 equal P = 1."""
    import paper_2111_00113_b200 as PK
    from inputs import start_block
    m, P = 96, 2
    n = m * m
    Om = start_block(n, 6, 3)
    v0 = np.random.default_rng(5).standard_normal(n)

    def fn_for(P_, kind):
        def fn(ctx, r):
            lo, hi = partition_rows("stencil2d", n, m, P_, r)
            A = PK.StencilOperator(2, m, 12.0, lo, hi)
            if kind == "block":
                return ctx.srr_eigs(A, np.ascontiguousarray(Om[lo:hi]), d=30, k=2, s=60, nev=5, zeta=8, seed=2,
                                    basis="block_chebyshev")
            return ctx.srr_eigs(A, v0[lo:hi].copy(), d=30, k=2, s=60, nev=5, zeta=8, seed=2, stabilize="always")
        return fn
    for kind in ("block", "stab"):
        ref = _run_ranks(1, fn_for(1, kind))[0]
        outs = _run_ranks(P, fn_for(P, kind))
        for o in outs:
            rel = np.abs(o["theta"] - ref["theta"]) / np.abs(ref["theta"])
            assert rel.max() <= 1e-10, (kind, rel)
            np.testing.assert_allclose(o["res_true"], ref["res_true"], rtol=1e-8)


def test_loopback_whitened_sgmres_matches_single_rank():
    """Whitening (O36) at P = 2: the whitening GEMM runs on each rank's rows, the column norms are all-reduced, the
    sketch update is replicated; same x as P = 1."""
    m, P = 32, 2
    n = m * m
    f = rhs_normal_local(n)
    kw = dict(d=45, k=2, s=120, zeta=8, seed=0, tol=1e-12, max_cycles=1, early_exit_factor=0.0, cond_tol=100.0,
              whiten=True)
    ref = _solve("stencil2d", m, n, 20.0, f, 1, kw)[0]
    outs = _solve("stencil2d", m, n, 20.0, f, P, kw)
    x = np.concatenate([o.x for o in outs])
    assert ref.info["flags"] & 32 and all(o.info["flags"] & 32 for o in outs)
    assert np.abs(x - ref.x).max() <= 1e-8 * np.abs(ref.x).max()


def rhs_normal_local(n):
    from inputs import rhs_normal
    return rhs_normal(n, 0)


@pytest.mark.parametrize("m,P", [(64, 2), (96, 4), (60, 3)])
def test_loopback_chebyshev_matrix_powers_2d(m, P):
    """2D Chebyshev basis with the matrix-powers launches (SKS_MPK_S columns per launch, ghost depth S + 1
    exchanged once per launch: SURVEY NEXT(1) 'depth-s halos') at P = 2, 3, 4 equals P = 1."""
    import os
    n = m * m
    f = np.random.default_rng(m + P).standard_normal(n)
    kw = dict(d=40, k=2, s=80, zeta=8, seed=4, tol=1e-10, max_cycles=2, basis="chebyshev")
    old = os.environ.get("SKS_MPK_S")
    os.environ["SKS_MPK_S"] = "4"
    try:
        ref = _solve("stencil2d", m, n, 15.0, f, 1, kw)[0]
        outs = _solve("stencil2d", m, n, 15.0, f, P, kw)
        plain = None
        os.environ["SKS_MPK_S"] = "0"
        plain = _solve("stencil2d", m, n, 15.0, f, 1, kw)[0]
    finally:
        if old is None:
            os.environ.pop("SKS_MPK_S", None)
        else:
            os.environ["SKS_MPK_S"] = old
    assert np.abs(ref.x - plain.x).max() <= 1e-10 * np.abs(plain.x).max()   # matrix powers = one step per launch
    x = np.concatenate([o.x for o in outs])
    assert all(o.info["columns"] == ref.info["columns"] for o in outs)
    assert np.abs(x - ref.x).max() <= 1e-10 * np.abs(ref.x).max()
