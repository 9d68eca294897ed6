"""Run ONE sGMRES solve of a BASELINE config on cuda:0 (for profiling under ncu)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2111_00113_b200 as P  # noqa: E402
from inputs import get_config, rhs_normal  # noqa: E402


def main(name="C3", cycles=None):
    cfg = get_config(name)
    ctx = P.Context(0)
    f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
    dim = 3 if cfg.op == "stencil3d" else 2
    A = P.StencilOperator(dim, cfg.m, cfg.beta)
    t = time.time()
    res = ctx.sgmres_solve(A, f, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol,
                           max_cycles=cycles or cfg.max_cycles)
    torch.cuda.synchronize()
    print(name, "wall", time.time() - t, "info", res.info)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C3", int(sys.argv[2]) if len(sys.argv) > 2 else None)
