"""Seeded input recipes.

* f ~ N(0,1): ``numpy.random.default_rng(seed).standard_normal(n)`` (O19).
* sRR start vector: ``default_rng(4).standard_normal(n)`` (O21; Alg. 2 P:1660 "randn").
* C4 CSR (O20): ``rng = default_rng(3)``; per row 16 DISTINCT columns uniform over
  j != i (draw in [0, n-1), shift past i, redraw duplicates); values
  ``standard_normal/4``; explicit diagonal 6.0; columns sorted; int32 indices;
  then f = ``rng.standard_normal(n)`` from the same stream.
* Row partition: contiguous blocks; for stencils whole grid lines (2D) / planes (3D).

No method arithmetic lives here.
"""
import numpy as np


def rhs_normal(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


def start_vector(n: int, seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal(n)


def start_block(n: int, b: int, seed: int) -> np.ndarray:
    """Start block Omega (n x b) of the block Krylov sRR ("drawn at random from a standard
    normal distribution"): column i is the i-th chunk of n draws of default_rng(seed) (F-ordered, so each
    column is contiguous)."""
    return np.asfortranarray(np.random.default_rng(seed).standard_normal((b, n)).T)


def random_csr_c4(n: int, seed: int = 3, nnz_off: int = 16, diag: float = 6.0):
    """Return (row_ptr int32[n+1], col_idx int32[nnz], val f64[nnz], f f64[n])."""
    rng = np.random.default_rng(seed)
    rows = np.arange(n, dtype=np.int64)[:, None]
    cols = rng.integers(0, n - 1, size=(n, nnz_off), dtype=np.int64)
    cols += (cols >= rows)
    # redraw duplicates until every row has nnz_off distinct off-diagonal columns
    while True:
        order = np.argsort(cols, axis=1, kind="stable")
        srt = np.take_along_axis(cols, order, axis=1)
        dup_sorted = np.zeros_like(srt, dtype=bool)
        dup_sorted[:, 1:] = srt[:, 1:] == srt[:, :-1]
        if not dup_sorted.any():
            break
        dup = np.zeros_like(dup_sorted)
        np.put_along_axis(dup, order, dup_sorted, axis=1)
        ri, ci = np.nonzero(dup)
        new = rng.integers(0, n - 1, size=ri.size, dtype=np.int64)
        new += (new >= ri)
        cols[ri, ci] = new
    vals = rng.standard_normal((n, nnz_off)) / 4.0
    f = rng.standard_normal(n)
    allc = np.concatenate([cols, rows], axis=1)
    allv = np.concatenate([vals, np.full((n, 1), diag)], axis=1)
    order = np.argsort(allc, axis=1, kind="stable")
    allc = np.take_along_axis(allc, order, axis=1)
    allv = np.take_along_axis(allv, order, axis=1)
    nnz_row = nnz_off + 1
    row_ptr = (np.arange(n + 1, dtype=np.int64) * nnz_row).astype(np.int32)
    return row_ptr, allc.reshape(-1).astype(np.int32), allv.reshape(-1).copy(), f


def partition_rows(kind: str, n: int, m: int, nranks: int, rank: int):
    """Contiguous row block [row_begin, row_end) of ``rank``.

    Stencils split whole y-lines (2D) or z-planes (3D) as evenly as possible;
    CSR splits rows as evenly as possible.  Mirrors ``sks_partition`` in the
    C-ABI (tests check the two agree).
    """
    if kind == "csr":
        unit, count = 1, n
    elif kind == "stencil2d":
        unit, count = m, m
    elif kind == "stencil3d":
        unit, count = m * m, m
    else:
        raise ValueError(kind)
    base, rem = divmod(count, nranks)
    lo = rank * base + min(rank, rem)
    hi = lo + base + (1 if rank < rem else 0)
    return lo * unit, hi * unit
