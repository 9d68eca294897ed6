"""C3 / C5 with the Chebyshev basis vs the BASELINE k-truncated Arnoldi basis:
device solve time, columns, true residual (median of 3 after a warm-up)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_00113_b200 as P
from inputs import get_config, rhs_normal, start_vector
ctx = P.Context(0)
for name in ("C3", "C2"):
    cfg = get_config(name)
    f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
    A = P.StencilOperator(3 if cfg.op == "stencil3d" else 2, cfg.m, cfg.beta)
    for basis in ("arnoldi", "chebyshev"):
        ts = []
        for r in range(4):
            res = ctx.sgmres_solve(A, f, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol,
                                   max_cycles=cfg.max_cycles, basis=basis)
            if r:
                ts.append(res.info["t_total_s"])
        print(json.dumps(dict(config=name, basis=basis, t_ms=statistics.median(ts) * 1e3, cycles=res.info["cycles"],
                              columns=res.info["columns_generated"], rel=res.info["rel_res_true"],
                              us_per_col=res.info["t_basis_s"] / res.info["columns_generated"] * 1e6)), flush=True)
