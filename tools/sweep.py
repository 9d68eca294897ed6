"""Run every BASELINE config once on cuda:0 (after one warm-up solve) and print one JSON line
each: device time, cycles, columns, true relative residual (sGMRES) or top Ritz values (sRR).
    python tools/sweep.py [C1 C2 ...]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2111_00113_b200 as P  # noqa: E402
from inputs import get_config, rhs_normal, start_vector, start_block, random_csr_c4  # noqa: E402


def main(names):
    ctx = P.Context(0)
    for name in names:
        cfg = get_config(name)
        t0 = time.time()
        if cfg.op == "csr":
            rp, ci, v, f = random_csr_c4(cfg.n, seed=cfg.seed)
            A = P.CsrOperator(rp, ci, v, cfg.n)
        else:
            A = P.StencilOperator(3 if cfg.op == "stencil3d" else 2, cfg.m, cfg.beta)
            f = rhs_normal(cfg.n, cfg.seed)
        tgen = time.time() - t0
        if cfg.method == "sgmres":
            ft = torch.from_numpy(f).cuda()
            kw = dict(d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol, max_cycles=cfg.max_cycles)
            ctx.sgmres_solve(A, ft, **kw)
            res = ctx.sgmres_solve(A, ft, **kw)
            i = res.info
            out = dict(config=name, t_total_ms=i["t_total_s"] * 1e3, t_basis_ms=i["t_basis_s"] * 1e3,
                       cycles=i["cycles"], columns=i["columns"], columns_generated=i["columns_generated"],
                       rel_res_true=i["rel_res_true"], us_per_column=i["t_basis_s"] / max(i["columns_generated"], 1) * 1e6,
                       launches=i["kernel_launches"])
        else:
            blk = cfg.method == "srr_block"
            v0 = torch.from_numpy(start_block(cfg.n, cfg.block, cfg.seed) if blk else start_vector(cfg.n, cfg.seed)).cuda()
            kw = dict(d=cfg.d, k=max(cfg.k, 1), s=cfg.s, nev=cfg.nev, zeta=cfg.zeta, seed=cfg.seed)
            if blk:
                kw["basis"] = "block_chebyshev"
            ctx.srr_eigs(A, v0, **kw)
            out_ = ctx.srr_eigs(A, v0, **kw)
            i = out_["info"]
            out = dict(config=name, t_total_ms=i["t_total_s"] * 1e3, t_basis_ms=i["t_basis_s"] * 1e3,
                       t_small_ms=i["t_small_s"] * 1e3, columns=i["columns"],
                       us_per_column=i["t_basis_s"] / max(i["columns"], 1) * 1e6,
                       theta=[complex(t).__repr__() for t in out_["theta"][:4]],
                       res_true=[float(r) for r in out_["res_true"][:4]], launches=i["kernel_launches"])
        out["host_gen_s"] = tgen
        print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5", "C5B"])
