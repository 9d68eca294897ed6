"""Compare hqr_dbg (GPU, after 1 sweep / to completion) with the Python emulation of the windowed
two-bulge sweep (/tmp/hq/kern2.py) and with numpy eigenvalues.  usage: python hqr_cmp.py make|check"""
import sys, struct, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.abspath(__file__)))
from scipy.linalg import hessenberg
n = 100
rng = np.random.default_rng(7)
H = hessenberg(rng.standard_normal((n, n)))
mask = np.triu(np.ones((n, n)), -1).astype(bool)
H = np.where(mask, H, 0.0)
an = np.abs(H).sum()
H = H / 2.0 ** np.floor(np.log2(an))
if sys.argv[1] == "make":
    with open('/root/repo/tools/micro/hqr_in.bin', 'wb') as f:
        f.write(struct.pack('i', n)); f.write(H.T.astype(np.float64).tobytes())   # column-major
    sys.exit(0)
def rd(p):
    b = open(p, 'rb').read()
    inf = struct.unpack('8i', b[:32]); o = np.frombuffer(b[32:], dtype=np.float64)
    return inf, o[:n * n].reshape(n, n).T, o[n * n:n * n + n], o[n * n + n:]
import hq_kern2 as kern2, hq_emul as emul
inf1, H1, _, _ = rd('/root/repo/gpurun_out/hqr_out1.bin')
nn = n - 1; l = 0
x = H[nn, nn]; y = H[nn - 1, nn - 1]; w = H[nn, nn - 1] * H[nn - 1, nn]
m = nn - 2
while m >= l:
    zz = H[m, m]; r = x - zz; s = y - zz
    p = (r * s - w) / H[m + 1, m] + H[m, m + 1]; q = H[m + 1, m + 1] - zz - r - s; r = H[m + 2, m + 1]
    s = abs(p) + abs(q) + abs(r); p /= s; q /= s; r /= s
    if m == l: break
    u = abs(H[m, m - 1]) * (abs(q) + abs(r)); v = abs(p) * (abs(H[m - 1, m - 1]) + abs(zz) + abs(H[m + 1, m + 1]))
    if u + v == v: break
    m -= 1
He = H.copy()
for i in range(m + 2, nn + 1):
    He[i, i - 2] = 0
    if i != m + 2: He[i, i - 3] = 0
kern2.windowed(He, l, m, nn, p, q, r, x, y, w)
print("m", m, "gpu info", inf1)
d = np.abs(np.where(mask, He - H1, 0))
print("1 sweep: max diff", d.max(), "at", np.unravel_index(d.argmax(), d.shape))
bad = np.argwhere(d > 1e-10)
print("first bad entries (row, col):", bad[:20].tolist())
inf, Hf, wr, wi = rd('/root/repo/gpurun_out/hqr_out.bin')
ev = np.sort_complex(wr + 1j * wi); ref = np.sort_complex(np.linalg.eigvals(H))
print("full:", inf, "eig err", np.abs(ev - ref).max())
