"""Sparse sign embedding S (Eq. sparse-map) -- oracle side.

Paper: S = (1/sqrt(s)) [s_1 ... s_n]; columns statistically independent; each
column has exactly zeta nonzeros, Steinhaus-distributed, "placed in uniformly
random coordinates".  Readings:
  O1  values +-1/sqrt(zeta) (BASELINE "values +-1/sqrt(8)"), so E||Sx||^2 = ||x||^2;
  O2  real Rademacher signs instead of complex Steinhaus;
  O3  zeta = 8 (BASELINE), not ceil(2 log(1+d));
  O5  the zeta distinct rows of column r are a uniformly random zeta-subset of
      {0..s-1} drawn by Floyd's algorithm from a counter-based hash, so S is never
      stored and CPU and GPU regenerate identical (row, sign) tables bit-exactly;
  O6/O7 seed = config seed; a fresh S per restart cycle c (key depends on c).

Hash specification (frozen; the CUDA side implements the same integer spec
independently, see include/sks.h):
  fmix64(z):  z ^= z>>30; z *= 0xBF58476D1CE4E5B9; z ^= z>>27;
              z *= 0x94D049BB133111EB; z ^= z>>31          (all mod 2^64)
  GAMMA = 0x9E3779B97F4A7C15
  key(seed, c)  = fmix64( fmix64(seed ^ 0x736B732D534B4554) + GAMMA*(c+1) )
  word(r, t)    = fmix64( key + GAMMA*(16*r + t) )          r = global row, 0-based
  draw u_t      = low 32 bits of word(r, t//2) if t even, else high 32 bits
  signs         = word(r, 8); sign_t = -1 if bit t set else +1
  Floyd, t = 0..zeta-1:  J = s - zeta + t;  v = (u_t * (J+1)) >> 32;
                         q_t = J if v in {q_0..q_{t-1}} else v
  S[q_t, r] = sign_t / sqrt(zeta)
Requires 1 <= zeta <= min(s, 16).
"""
import numpy as np
import scipy.sparse as sp

_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_DOMAIN = np.uint64(0x736B732D534B4554)
_MASK32 = np.uint64(0xFFFFFFFF)


def fmix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z ^ (z >> np.uint64(30))
        z = z * _M1
        z = z ^ (z >> np.uint64(27))
        z = z * _M2
        z = z ^ (z >> np.uint64(31))
    return z


def sketch_key(seed: int, cycle: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k0 = fmix64(np.array([np.uint64(seed) ^ _DOMAIN], dtype=np.uint64))
        k = fmix64(k0 + _GAMMA * np.uint64(cycle + 1))
    return np.uint64(k[0])


def floyd(draws, s: int):
    """Floyd's algorithm: draws[t] in [0, s-zeta+t] -> ordered zeta-subset of
    {0..s-1}, uniform over subsets when the draws are uniform and independent."""
    zeta = len(draws)
    q = np.empty((np.asarray(draws[0]).size, zeta), dtype=np.int64)
    for t in range(zeta):
        J = s - zeta + t
        v = np.asarray(draws[t], dtype=np.int64).reshape(-1)
        if t > 0:
            taken = (q[:, :t] == v[:, None]).any(axis=1)
            v = np.where(taken, J, v)
        q[:, t] = v
    return q


def sketch_table(rows, s: int, zeta: int, seed: int, cycle: int = 0):
    """(q, sign) tables, shapes (len(rows), zeta): q int64 in [0,s), sign in {+1,-1}."""
    if not (1 <= zeta <= min(s, 16)):
        raise ValueError("need 1 <= zeta <= min(s, 16)")
    rows = np.asarray(rows, dtype=np.uint64)
    key = sketch_key(seed, cycle)
    nr = rows.size
    q = np.empty((nr, zeta), dtype=np.int64)
    with np.errstate(over="ignore"):
        base = key + _GAMMA * (np.uint64(16) * rows)
        words = [fmix64(base + _GAMMA * np.uint64(t)) for t in range((zeta + 1) // 2)]
        sword = fmix64(base + _GAMMA * np.uint64(8))
    draws = []
    for t in range(zeta):
        w = words[t // 2]
        u = (w & _MASK32) if t % 2 == 0 else (w >> np.uint64(32))
        J = s - zeta + t
        draws.append(((u * np.uint64(J + 1)) >> np.uint64(32)).astype(np.int64))
    q[:] = floyd(draws, s)
    bits = ((sword[:, None] >> np.arange(zeta, dtype=np.uint64)[None, :]) & np.uint64(1))
    sign = np.where(bits.astype(bool), -1.0, 1.0)
    return q, sign


def sketch_matrix(n: int, s: int, zeta: int, seed: int, cycle: int = 0,
                  row_begin: int = 0, row_end: int = None, chunk: int = 1 << 20):
    """S restricted to global columns [row_begin, row_end) as scipy CSR (s x n_local)."""
    if row_end is None:
        row_end = n
    nl = row_end - row_begin
    data, ri, ci = [], [], []
    scale = 1.0 / np.sqrt(float(zeta))
    for lo in range(row_begin, row_end, chunk):
        hi = min(row_end, lo + chunk)
        rows = np.arange(lo, hi, dtype=np.int64)
        q, sign = sketch_table(rows, s, zeta, seed, cycle)
        data.append((sign * scale).ravel())
        ri.append(q.ravel())
        ci.append(np.repeat(rows - row_begin, zeta))
    data = np.concatenate(data) if data else np.zeros(0)
    ri = np.concatenate(ri) if ri else np.zeros(0, dtype=np.int64)
    ci = np.concatenate(ci) if ci else np.zeros(0, dtype=np.int64)
    return sp.csr_matrix((data, (ri, ci)), shape=(s, nl))


def sketch_apply(M, s: int, zeta: int, seed: int, cycle: int = 0, row_begin: int = 0,
                 n: int = None):
    """S M for M of shape (n_local,) or (n_local, c); rows are global [row_begin, ...)."""
    M = np.asarray(M, dtype=np.float64)
    nl = M.shape[0]
    if n is None:
        n = row_begin + nl
    S = sketch_matrix(n, s, zeta, seed, cycle, row_begin, row_begin + nl)
    return S @ M
