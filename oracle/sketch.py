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


# ---------------------------------------------------------------- SRFT
# Eq. (SRFT): S = sqrt(n/s) D F E with E a random diagonal of unit-modulus entries, F
# the unitary DFT and D a random projector onto s coordinates; the paper's experiments use
# F = DCT2, a real orthonormal transform.  Readings (O32): real
# Rademacher E (as O2), F = orthonormal DCT-II, the s coordinates drawn by Floyd's algorithm
# (uniform s-subset of {0..n-1}) in draw order = sketch row order, a fresh S per cycle.
# Hash specification (the CUDA driver implements the same integer spec independently):
#   key(seed, c) = fmix64( fmix64(seed ^ 0x5352465444435432) + GAMMA*(c+1) )
#   sign(r)      = -1 if bit 0 of fmix64(key + GAMMA*(2r+1)) else +1        r = 0..n-1
#   Floyd, t = 0..s-1:  u_t = low 32 bits of fmix64(key + GAMMA*(2t+2));  J = n - s + t;
#                       v = (u_t * (J+1)) >> 32;  q_t = J if v in {q_0..q_{t-1}} else v
#   (S x)_t = sqrt(n/s) * DCT2_ortho(E x)[q_t]
_SRFT_DOMAIN = np.uint64(0x5352465444435432)


def srft_key(seed: int, cycle: int) -> np.uint64:
    with np.errstate(over="ignore"):
        k0 = fmix64(np.array([np.uint64(seed) ^ _SRFT_DOMAIN], dtype=np.uint64))
        k = fmix64(k0 + _GAMMA * np.uint64(cycle + 1))
    return np.uint64(k[0])


def srft_signs(n: int, seed: int, cycle: int = 0):
    key = srft_key(seed, cycle)
    r = np.arange(n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        w = fmix64(key + _GAMMA * (np.uint64(2) * r + np.uint64(1)))
    return np.where((w & np.uint64(1)).astype(bool), -1.0, 1.0)


def srft_rows(n: int, s: int, seed: int, cycle: int = 0):
    """The s sampled DCT coordinates, in sketch-row order (Floyd, plain loop)."""
    if not (1 <= s <= n < 2 ** 32):
        raise ValueError("need 1 <= s <= n < 2^32")
    key = srft_key(seed, cycle)
    t = np.arange(s, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u = fmix64(key + _GAMMA * (np.uint64(2) * t + np.uint64(2))) & _MASK32
    q = []
    taken = set()
    for i in range(s):
        J = n - s + i
        v = int((int(u[i]) * (J + 1)) >> 32)
        if v in taken:
            v = J
        taken.add(v)
        q.append(v)
    return np.array(q, dtype=np.int64)


def srft_apply(M, s: int, seed: int, cycle: int = 0):
    """S M for the SRFT of Eq. (SRFT) with F = orthonormal DCT-II."""
    from scipy.fft import dct
    M = np.asarray(M, dtype=np.float64)
    n = M.shape[0]
    E = srft_signs(n, seed, cycle)
    Y = dct(E.reshape((n,) + (1,) * (M.ndim - 1)) * M, type=2, norm="ortho", axis=0)
    return np.sqrt(n / s) * Y[srft_rows(n, s, seed, cycle)]


class SRFT:
    """S as an operator (S @ x, S @ M) for the sGMRES / sRR oracles."""

    def __init__(self, n: int, s: int, seed: int, cycle: int = 0):
        self.n, self.s, self.seed, self.cycle = n, s, seed, cycle
        self.shape = (s, n)

    def __matmul__(self, M):
        return srft_apply(M, self.s, self.seed, self.cycle)
