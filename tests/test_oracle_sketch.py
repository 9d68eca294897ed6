"""Pins of oracle/sketch.py (sparse sign map) against what the paper fixes.

* every column has exactly zeta nonzeros at distinct rows, values +-1/sqrt(zeta)
  ("exactly zeta nonzero entries", O1);
* Floyd's step yields every zeta-subset equally often (exhaustive enumeration of
  the draw space -- brute force on tiny inputs);
* row / sign marginals uniform (chi-square), columns of different cycles differ;
* subspace-embedding distortion (Def. P:527-536) near sqrt(d/s) = 1/sqrt(2) at s = 2d
  ("s = d/eps^2"; "eps = 1/sqrt(2)");
* E||Sx||^2 = ||x||^2 (isotropy of the +-1/sqrt(zeta) scaling, O1);
* S M equals the dense materialised product.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle as O
from oracle.sketch import floyd

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_columns_exact_zeta_distinct():
    n, s, z = 20000, 120, 8
    q, sign = O.sketch_table(np.arange(n), s, z, seed=0, cycle=0)
    assert q.min() >= 0 and q.max() < s
    srt = np.sort(q, axis=1)
    assert np.all(np.diff(srt, axis=1) > 0)
    assert set(np.unique(sign)) == {-1.0, 1.0}
    S = O.sketch_matrix(n, s, z, seed=0).toarray()
    nnz = (S != 0).sum(axis=0)
    assert np.all(nnz == z)
    assert np.allclose(np.abs(S[S != 0]), 1 / np.sqrt(8.0), rtol=0, atol=0)


def test_floyd_exhaustive_uniform():
    # every (draw_0 in [0,s-z], draw_1 in [0,s-z+1], ...) combination; each subset
    # must be produced equally often (Floyd's theorem), i.e. uniform over subsets.
    for s, z in [(5, 2), (6, 3), (7, 3), (5, 5)]:
        ranges = [range(s - z + t + 1) for t in range(z)]
        combos = np.array(list(itertools.product(*ranges)))
        q = floyd([combos[:, t] for t in range(z)], s)
        assert np.all(np.diff(np.sort(q, axis=1), axis=1) > 0)
        keys = [tuple(sorted(r)) for r in q.tolist()]
        counts = {}
        for k in keys:
            counts[k] = counts.get(k, 0) + 1
        from math import comb
        assert len(counts) == comb(s, z)
        assert len(set(counts.values())) == 1


def test_marginals_chi_square():
    n, s, z = 60000, 64, 8
    q, sign = O.sketch_table(np.arange(n), s, z, seed=7, cycle=3)
    counts = np.bincount(q.ravel(), minlength=s)
    exp = n * z / s
    chi2 = ((counts - exp) ** 2 / exp).sum()
    assert chi2 < s + 6 * np.sqrt(2 * s)       # dof = s-1, ~6 sigma
    assert abs(sign.mean()) < 6 / np.sqrt(sign.size)
    # joint law: every zeta-subset equally likely (hash + Floyd), s=12, zeta=3
    from math import comb
    n2, s2, z2 = 200000, 12, 3
    q2, _ = O.sketch_table(np.arange(n2), s2, z2, seed=1, cycle=0)
    srt = np.sort(q2, axis=1)
    code = (srt[:, 0] * s2 + srt[:, 1]) * s2 + srt[:, 2]
    _, cnt = np.unique(code, return_counts=True)
    ns = comb(s2, z2)
    assert cnt.size == ns
    e = n2 / ns
    assert ((cnt - e) ** 2 / e).sum() < ns + 6 * np.sqrt(2 * ns)


def test_deterministic_and_fresh_per_cycle():
    rows = np.arange(1000, 3000)
    a = O.sketch_table(rows, 600, 8, seed=2, cycle=0)
    b = O.sketch_table(rows, 600, 8, seed=2, cycle=0)
    c = O.sketch_table(rows, 600, 8, seed=2, cycle=1)
    d = O.sketch_table(rows, 600, 8, seed=3, cycle=0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert (a[0] != c[0]).mean() > 0.9 and (a[0] != d[0]).mean() > 0.9
    # the table of a row does not depend on which other rows are requested
    e = O.sketch_table(rows[500:600], 600, 8, seed=2, cycle=0)
    assert np.array_equal(e[0], a[0][500:600])


@pytest.mark.parametrize("n,d", [(4096, 20), (20000, 60)])
def test_subspace_embedding_distortion(n, d):
    s, z = 2 * d, 8
    gold = json.load(open(os.path.join(GOLD, "paper_bounds.json")))
    rng = np.random.default_rng(11)
    eps = []
    for trial in range(8):
        Q, _ = np.linalg.qr(rng.standard_normal((n, d)))
        SQ = O.sketch_apply(Q, s, z, seed=100 + trial)
        sv = np.linalg.svd(SQ, compute_uv=False)
        eps.append(max(sv.max() - 1, 1 - sv.min()))
    eps = np.array(eps)
    # Gaussian-like behaviour: sqrt(d/s) = 1/sqrt(2); SURVEY thresholds
    assert abs(eps.mean() - gold["eps_at_s_2d"]) < 0.06
    assert eps.max() <= 0.80
    # and therefore the sGMRES sandwich factor (1+eps)/(1-eps) stays near the paper's "< 6"
    assert ((1 + eps.mean()) / (1 - eps.mean())) < gold["sandwich_factor_max"] * 1.2


def test_isotropy_expected_norm():
    n, s, z = 3000, 50, 8
    rng = np.random.default_rng(5)
    x = rng.standard_normal(n)
    vals = [np.linalg.norm(O.sketch_apply(x, s, z, seed=sd)) ** 2 for sd in range(200)]
    assert abs(np.mean(vals) / np.dot(x, x) - 1) < 0.03


def test_apply_equals_dense_and_linear():
    n, s, z = 700, 40, 8
    rng = np.random.default_rng(1)
    M = rng.standard_normal((n, 5))
    S = O.sketch_matrix(n, s, z, seed=4, cycle=2).toarray()
    SM = O.sketch_apply(M, s, z, seed=4, cycle=2)
    np.testing.assert_allclose(SM, S @ M, rtol=1e-13, atol=1e-13)
    # dense S built by brute force from the table (rows -> columns)
    q, sign = O.sketch_table(np.arange(n), s, z, seed=4, cycle=2)
    Sb = np.zeros((s, n))
    for r in range(n):
        for t in range(z):
            Sb[q[r, t], r] += sign[r, t] / np.sqrt(z)
    assert np.array_equal(Sb, S)
    # row-block restriction: global row indices are what matter
    part = O.sketch_apply(M[300:], s, z, seed=4, cycle=2, row_begin=300, n=n)
    np.testing.assert_allclose(part, S[:, 300:] @ M[300:], rtol=1e-13, atol=1e-13)
