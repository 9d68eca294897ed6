"""Tiny invocations of every kernel family of libsks, for compute-sanitizer (racecheck / synccheck / memcheck):

  3D z-march TMA step kernel (m = 24), 2D tiled TMA step (m = 64), 2D y-march TMA step (m = 1024, few columns),
  the odd-m plain step kernels, CSR SpMV + orthogonalisation, the sketch plan / gather / reduce, BCGS2 + CholQR
  panels, assembly, sRR (Hessenberg/Francis QR, inverse iteration, Ritz vectors), the stabilised sRR (cooperative
  Jacobi SVD + Hessenberg reduction), the Chebyshev basis and the SRFT sketch.

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py
Exit code 0 and "ALL CASES RAN" on success (numerical results are checked by the pytest suite, not here).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_00113_b200 as P  # noqa: E402
from inputs import random_csr_c4  # noqa: E402


def main():
    ctx = P.Context(0)
    rng = np.random.default_rng(7)
    cases = [
        ("3d-zm", P.StencilOperator(3, 24, 30.0), dict(d=12, k=2, s=24)),
        ("3d-odd", P.StencilOperator(3, 15, 30.0), dict(d=8, k=2, s=16)),
        ("2d-tma", P.StencilOperator(2, 64, 20.0), dict(d=12, k=4, s=24)),
        ("2d-odd", P.StencilOperator(2, 33, 20.0), dict(d=8, k=2, s=16)),
        ("2d-ym", P.StencilOperator(2, 1024, 10.0), dict(d=5, k=2, s=10)),
    ]
    for name, A, kw in cases:
        f = torch.from_numpy(rng.standard_normal(A.n_global)).cuda()
        r = ctx.sgmres_solve(A, f, zeta=8, seed=1, tol=1e-8, max_cycles=2, **kw)
        print(name, r.info["columns_generated"], r.info["rel_res_true"], flush=True)
    rp, ci, v, fc = random_csr_c4(4000, seed=3)
    r = ctx.sgmres_solve(P.CsrOperator(rp, ci, v, 4000), torch.from_numpy(fc).cuda(), d=10, k=2, s=20, zeta=8,
                         seed=3, max_cycles=2)
    print("csr", r.info["columns_generated"], r.info["rel_res_true"], flush=True)
    A2 = P.StencilOperator(2, 64, 10.0)
    v0 = rng.standard_normal(A2.n_global)
    for stab in ("off", "always"):
        o = ctx.srr_eigs(A2, v0, d=24, k=2, s=48, nev=4, zeta=8, seed=4, stabilize=stab, want_vectors=True)
        print("srr", stab, o["theta"][:2], flush=True)
    f2 = torch.from_numpy(rng.standard_normal(A2.n_global)).cuda()
    r = ctx.sgmres_solve(A2, f2, d=12, k=2, s=24, zeta=8, seed=1, max_cycles=2, basis="chebyshev")
    print("cheb", r.info["columns_generated"], flush=True)
    r = ctx.sgmres_solve(A2, f2, d=12, k=2, s=24, zeta=8, seed=1, max_cycles=2, sketch="srft")
    print("srft", r.info["columns_generated"], flush=True)
    torch.cuda.synchronize()
    ctx.close()
    print("ALL CASES RAN")


if __name__ == "__main__":
    main()
