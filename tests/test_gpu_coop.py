"""GPU parity of the cooperative small-problem basis kernels (stencil_coop.cu; opt-in, measured slower than the
per-column launches at C2 -- profiles/r02/coop_ab_r02.txt) against the oracle, through the C ABI:

  * SKS_COOP_MAXN:  a batch of columns per cooperative launch, two grid barriers per column (2D and 3D);
  * SKS_COOP1_MAXN: one grid barrier per column, a ring of k + 1 columns in shared memory and one recomputed halo
                    line per side (2D, even m; ragged last CTA when L does not divide m).

Same bar as tests/test_gpu_parity.py: residual within 2x of the oracle's, equal cycles / columns, the r_est history
to 1e-6, Ritz values to 1e-8.
"""
import numpy as np
import pytest

import oracle as O
from inputs import rhs_normal, start_vector

pytestmark = pytest.mark.gpu

KERNELS = {"coop": "SKS_COOP_MAXN", "coop1": "SKS_COOP1_MAXN"}


@pytest.fixture(scope="module")
def ctx():
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200 import build
    build.build()
    c = P.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("kern", ["coop", "coop1"])
@pytest.mark.parametrize("dim,m,beta,d,k,basis", [(2, 64, 20.0, 60, 2, "arnoldi"), (2, 130, 50.0, 50, 4, "arnoldi"),
                                                  (2, 96, 20.0, 60, 2, "chebyshev"), (2, 32, 20.0, 60, 2, "arnoldi"),
                                                  (3, 24, 30.0, 40, 2, "arnoldi")])
def test_coop_sgmres_matches_oracle(ctx, monkeypatch, kern, dim, m, beta, d, k, basis):
    import paper_2111_00113_b200 as P
    if kern == "coop1" and dim == 3:
        pytest.skip("the one-barrier kernel is 2D only")
    monkeypatch.setenv(KERNELS[kern], str(10 ** 7))
    n = m ** dim
    f = rhs_normal(n, 3)
    Ao = O.stencil_matrix(dim, m, beta)
    cheb = O.spectral_box(dim, m, beta) if basis == "chebyshev" else None
    res = ctx.sgmres_solve(P.StencilOperator(dim, m, beta), f, d=d, k=k, s=2 * d, seed=3, tol=1e-8, max_cycles=6,
                           basis=basis)
    orc = O.sgmres_solve(lambda x: Ao @ x, f, d, 2 if basis == "chebyshev" else k, 2 * d, 8, 3, tol=1e-8,
                         max_cycles=6, cheb=cheb)
    rel_gpu = np.linalg.norm(f - Ao @ res.x) / np.linalg.norm(f)
    assert rel_gpu <= 2 * orc["rel_res_true"] and orc["rel_res_true"] <= 2 * rel_gpu
    assert res.info["cycles"] == orc["cycles"] and res.info["columns"] == orc["columns"]
    np.testing.assert_allclose(res.hist, orc["hist_est"], rtol=1e-6)


@pytest.mark.parametrize("kern", ["coop", "coop1"])
def test_coop_srr_matches_oracle(ctx, monkeypatch, kern):
    import paper_2111_00113_b200 as P
    monkeypatch.setenv(KERNELS[kern], str(10 ** 7))
    m, beta, d = 48, 10.0, 60
    v0 = start_vector(m * m, 4)
    out = ctx.srr_eigs(P.StencilOperator(2, m, beta), v0, d=d, k=2, s=2 * d, nev=5, seed=4)
    Ao = O.stencil_matrix(2, m, beta)
    ref = O.srr_eigs(lambda v: Ao @ v, v0, d, 2, 2 * d, 8, 4, 5)
    for t in out["theta"]:
        assert np.min(np.abs(ref["theta_all"] - t) / np.abs(t)) <= 1e-8


def test_coop1_equals_per_column_launches(ctx, monkeypatch):
    """The recomputed halo lines equal the neighbours' own lines bit for bit, so the one-barrier kernel produces the
    per-column launches' basis up to the kernels' different (fixed) summation orders."""
    import paper_2111_00113_b200 as P
    m = 256
    f = rhs_normal(m * m, 5)
    kw = dict(d=40, k=4, s=80, seed=5, tol=1e-12, max_cycles=1, early_exit_factor=0.0)
    monkeypatch.setenv("SKS_COOP1_MAXN", "0")
    a = ctx.sgmres_solve(P.StencilOperator(2, m, 20.0), f, **kw)
    monkeypatch.setenv("SKS_COOP1_MAXN", str(10 ** 7))
    b = ctx.sgmres_solve(P.StencilOperator(2, m, 20.0), f, **kw)
    assert b.info["kernel_launches"] < a.info["kernel_launches"]  # the batches ran as cooperative launches
    assert np.abs(a.x - b.x).max() <= 1e-10 * np.abs(a.x).max()
    np.testing.assert_allclose(a.hist, b.hist, rtol=1e-9)
