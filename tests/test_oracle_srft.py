"""Pins of the oracle's SRFT sketch (Eq. SRFT P:631-638 with F = DCT2 as in the paper's experiments,
P:2041-2043; reading O32), checked against definitions other than the implementation:

  * the explicit DCT-II matrix written out from its textbook formula (not scipy's transform):
    S = sqrt(n/s) P C E column by column;
  * s = n: S = C E is orthogonal (S^T S = I, norms preserved);
  * the sampled coordinates are distinct and uniform (chi^2 over seeds), the signs balanced;
  * E ||S x||^2 = ||x||^2 over independent draws, and the subspace-embedding distortion at s = 2d
    is of the size the theory predicts (like the sparse map's).
"""
import numpy as np

import oracle as O


def _dct2_matrix(n):
    k = np.arange(n)[:, None]
    j = np.arange(n)[None, :]
    C = np.sqrt(2.0 / n) * np.cos(np.pi * k * (2 * j + 1) / (2 * n))
    C[0, :] /= np.sqrt(2.0)
    return C


def test_matches_the_explicit_dct_matrix():
    n, s = 48, 12
    for seed, cycle in [(0, 0), (3, 2)]:
        S = O.srft_apply(np.eye(n), s, seed, cycle)
        E = np.diag(O.srft_signs(n, seed, cycle))
        P = np.eye(n)[O.srft_rows(n, s, seed, cycle)]
        ref = np.sqrt(n / s) * P @ _dct2_matrix(n) @ E
        assert np.abs(S - ref).max() <= 1e-13


def test_full_sampling_is_orthogonal():
    n = 64
    S = O.srft_apply(np.eye(n), n, 5, 1)
    assert np.abs(S.T @ S - np.eye(n)).max() <= 1e-13
    x = np.random.default_rng(1).standard_normal(n)
    assert abs(np.linalg.norm(O.srft_apply(x, n, 5, 1)) - np.linalg.norm(x)) <= 1e-13 * np.linalg.norm(x)


def test_rows_distinct_uniform_and_signs_balanced():
    n, s, trials = 20, 5, 4000
    counts = np.zeros(n)
    for seed in range(trials):
        q = O.srft_rows(n, s, seed, 0)
        assert len(set(q.tolist())) == s and q.min() >= 0 and q.max() < n
        counts[q] += 1
    expect = trials * s / n
    chi2 = ((counts - expect) ** 2 / expect).sum()
    assert chi2 < 45.0                                    # dof 19: p ~ 1e-3
    sg = O.srft_signs(200_000, 7, 3)
    assert abs(sg.mean()) < 0.01 and set(np.unique(sg)) == {-1.0, 1.0}
    assert not np.array_equal(O.srft_rows(1000, 50, 1, 0), O.srft_rows(1000, 50, 1, 1))   # fresh per cycle


def test_norm_preserved_in_expectation_and_embedding_distortion():
    rng = np.random.default_rng(2)
    n, s = 4096, 128
    x = rng.standard_normal(n)
    r = [np.linalg.norm(O.srft_apply(x, s, seed, 0)) ** 2 for seed in range(200)]
    assert abs(np.mean(r) / np.dot(x, x) - 1.0) < 0.03
    d = 32                                               # s = 4d: distortion ~ sqrt(d/s) = 0.5
    Q, _ = np.linalg.qr(rng.standard_normal((n, d)))
    sv = np.linalg.svd(O.srft_apply(Q, 2 * d * 2, 9, 0), compute_uv=False)
    assert sv.max() < 1.7 and sv.min() > 0.3
