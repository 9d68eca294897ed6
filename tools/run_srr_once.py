"""Run sRR on a BASELINE sRR config (default C5) on cuda:0: `reps` calls (for profiling under ncu
or the hqr diagnostics, SKS_DEBUG_HQR=1)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_00113_b200 as P  # noqa: E402
from inputs import get_config, start_vector, start_block  # noqa: E402


def main(name="C5", reps=1, stabilize="off"):
    cfg = get_config(name)
    ctx = P.Context(0)
    blk = cfg.method == "srr_block"
    v0 = (torch.from_numpy(start_block(cfg.n, cfg.block, cfg.seed)) if blk
          else torch.from_numpy(start_vector(cfg.n, cfg.seed))).cuda()
    A = P.StencilOperator(2, cfg.m, cfg.beta)
    kw = dict(basis="block_chebyshev") if blk else {}
    for _ in range(reps):
        out = ctx.srr_eigs(A, v0, d=cfg.d, k=max(cfg.k, 1), s=cfg.s, nev=cfg.nev, zeta=cfg.zeta, seed=cfg.seed,
                           stabilize=stabilize, **kw)
    torch.cuda.synchronize()
    i = out["info"]
    print(name, "stabilize", stabilize, "rank", i["rank"], "t_total_ms", i["t_total_s"] * 1e3, "t_basis_ms",
          i["t_basis_s"] * 1e3, "bytes_basis_GB", i["bytes_basis"] / 1e9, "t_small_ms",
          i["t_small_s"] * 1e3, "theta", out["theta"][:3], "res_true", out["res_true"][:3], flush=True)
    ctx.close()


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "C5", int(sys.argv[2]) if len(sys.argv) > 2 else 1,
         sys.argv[3] if len(sys.argv) > 3 else "off")
