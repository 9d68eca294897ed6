"""ELL vs CSR SpMV paths (csr.cu): the ELL copy is built at set-up for near-uniform rows
(longest <= 32 and <= 1.25 x average + 1) and SKS_CSR_ELL=0 keeps the CSR kernel.  Both paths must equal the oracle's
SpMV and give the same sGMRES iterate; a matrix with skewed row lengths must take the CSR path and still be exact.
The switch is read at every operator set-up, so both paths run in one process."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

import oracle as O
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


def _with_ell(flag, fn):
    old = os.environ.get("SKS_CSR_ELL")
    os.environ["SKS_CSR_ELL"] = flag
    try:
        return fn()
    finally:
        if old is None:
            del os.environ["SKS_CSR_ELL"]
        else:
            os.environ["SKS_CSR_ELL"] = old


@pytest.mark.parametrize("n", [20_000, 33_333])
def test_ell_and_csr_apply_equal_oracle(ctx, n):
    import paper_2111_00113_b200 as P
    rp, ci, v, f = random_csr_c4(n, seed=5)
    ref = O.csr_matrix(rp, ci, v, n) @ f
    for flag in ("1", "0"):
        y = _with_ell(flag, lambda: ctx.apply_operator(P.CsrOperator(rp, ci, v, n), f))
        assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref), flag


def test_ell_and_csr_sgmres_agree(ctx):
    import paper_2111_00113_b200 as P
    n = 30_000
    rp, ci, v, f = random_csr_c4(n, seed=3)
    kw = dict(d=40, k=2, s=80, seed=3, tol=1e-8, max_cycles=3)
    r1 = _with_ell("1", lambda: ctx.sgmres_solve(P.CsrOperator(rp, ci, v, n), f, **kw))
    r0 = _with_ell("0", lambda: ctx.sgmres_solve(P.CsrOperator(rp, ci, v, n), f, **kw))
    assert r1.info["columns_generated"] == r0.info["columns_generated"]
    assert np.linalg.norm(r1.x - r0.x) <= 1e-10 * np.linalg.norm(r0.x)
    A = O.csr_matrix(rp, ci, v, n)
    for r in (r0, r1):
        assert np.linalg.norm(A @ r.x - f) / np.linalg.norm(f) <= 1e-8


def test_skewed_rows_take_csr_and_stay_exact(ctx):
    import paper_2111_00113_b200 as P
    n = 12_000
    rng = np.random.default_rng(11)
    lens = np.where(rng.random(n) < 0.01, 200, 3)  # 1% of the rows are 200 long: not ELL-shaped
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, n, size=rows.size)
    A = sp.csr_matrix((rng.standard_normal(rows.size) / 4, (rows, cols)), shape=(n, n)) + 6.0 * sp.identity(n)
    A = A.tocsr()
    A.sort_indices()
    x = rng.standard_normal(n)
    y = ctx.apply_operator(P.CsrOperator(A.indptr.astype(np.int32), A.indices.astype(np.int32), A.data, n), x)
    ref = O.csr_matrix(A.indptr, A.indices, A.data, n) @ x
    assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)
