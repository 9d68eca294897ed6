"""Bitwise run-to-run determinism of the GPU path (every reduction is a fixed-order sum of per-CTA partials; the
sketch plan orders its buckets without atomics; no floating-point atomics anywhere).  A data race or an
unsynchronised shared-memory hand-off (TMA/mbarrier pipelines, warp-specialised step kernel, PDL) shows up as
run-to-run differences, so this doubles as the race check that compute-sanitizer cannot provide on this pool
(profiles/r02/compute_sanitizer_r02a.txt).  Configurations cover the 3D z-march kernel (even m), the 2D tiled and
y-march kernels, the odd-m plain kernels, CSR, and sRR."""
import numpy as np
import pytest

from inputs import random_csr_c4

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200 import build
    build.build()
    c = P.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("dim,m,k,d", [(3, 64, 2, 40), (3, 33, 2, 20), (2, 256, 4, 60), (2, 1024, 2, 24),
                                       (2, 65, 2, 30)])
def test_sgmres_bitwise_repeatable(ctx, dim, m, k, d):
    import torch
    import paper_2111_00113_b200 as P
    A = P.StencilOperator(dim, m, 20.0)
    f = torch.from_numpy(np.random.default_rng(m).standard_normal(m ** dim)).cuda()
    runs = [ctx.sgmres_solve(A, f, d=d, k=k, s=2 * d, zeta=8, seed=3, tol=1e-10, max_cycles=2) for _ in range(3)]
    x0 = runs[0].x.cpu().numpy()
    for r in runs[1:]:
        assert np.array_equal(r.x.cpu().numpy(), x0)
        assert np.array_equal(r.hist, runs[0].hist)
        assert r.info["columns_generated"] == runs[0].info["columns_generated"]


def test_csr_and_srr_bitwise_repeatable(ctx):
    import torch
    import paper_2111_00113_b200 as P
    rp, ci, v, f = random_csr_c4(20000, seed=3)
    A = P.CsrOperator(rp, ci, v, 20000)
    ft = torch.from_numpy(f).cuda()
    r1 = ctx.sgmres_solve(A, ft, d=20, k=2, s=40, zeta=8, seed=3)
    r2 = ctx.sgmres_solve(A, ft, d=20, k=2, s=40, zeta=8, seed=3)
    assert np.array_equal(r1.x.cpu().numpy(), r2.x.cpu().numpy())
    S = P.StencilOperator(2, 256, 10.0)
    v0 = np.random.default_rng(4).standard_normal(256 * 256)
    o1 = ctx.srr_eigs(S, v0, d=60, k=2, s=120, nev=6, zeta=8, seed=4)
    o2 = ctx.srr_eigs(S, v0, d=60, k=2, s=120, nev=6, zeta=8, seed=4)
    assert np.array_equal(o1["theta"], o2["theta"]) and np.array_equal(o1["res_true"], o2["res_true"])
