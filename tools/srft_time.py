"""C3 / C5 with the SRFT sketch (reading O32) vs the sparse sign map: device solve time,
cycles, columns, residual (median of 3 after a warm-up)."""
import os, sys, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_00113_b200 as P
from inputs import get_config, rhs_normal, start_vector
ctx = P.Context(0)
cfg = get_config("C3")
f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
A = P.StencilOperator(3, cfg.m, cfg.beta)
for sk in ("sparse", "srft"):
    ts = []
    for r in range(4):
        res = ctx.sgmres_solve(A, f, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol,
                               max_cycles=cfg.max_cycles, sketch=sk)
        if r:
            ts.append(res.info["t_total_s"])
    print(json.dumps(dict(config="C3", sketch=sk, t_ms=statistics.median(ts) * 1e3, cycles=res.info["cycles"],
                          columns=res.info["columns_generated"], rel=res.info["rel_res_true"])), flush=True)
cfg = get_config("C5")
v0 = torch.from_numpy(start_vector(cfg.n, cfg.seed)).cuda()
A = P.StencilOperator(2, cfg.m, cfg.beta)
for sk in ("sparse", "srft"):
    ts = []
    for r in range(3):
        out = ctx.srr_eigs(A, v0, d=cfg.d, k=cfg.k, s=cfg.s, nev=cfg.nev, zeta=cfg.zeta, seed=cfg.seed, sketch=sk)
        if r:
            ts.append(out["info"]["t_total_s"])
    print(json.dumps(dict(config="C5", sketch=sk, t_ms=statistics.median(ts) * 1e3,
                          theta0=str(out["theta"][0]), res0=float(out["res_true"][0]))), flush=True)
