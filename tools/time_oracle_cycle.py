"""Measure the CPU oracle (as it stands, never tuned) on ONE FULL restart cycle of a BASELINE config at its real
sizes (C3: n = 4,096,000, d = 300, k = 2, s = 600, zeta = 8): residual, k-truncated Arnoldi basis of d columns,
sparse sketch of AB, thin QR, the r_est history, the LS solve, the update of x and the true residual -- exactly
oracle.sgmres_cycle (Alg. 1).  Timed single-threaded and with all host cores (threadpoolctl limits the
BLAS pools; scipy's sparse products are single-threaded either way).  Prints one JSON line with the CPU model and
the core count, so bench.py's bounded-sample extrapolation (cpu_baseline) can be checked against a measured cycle.

    python tools/time_oracle_cycle.py [--config C3] [--modes 1,all]
"""
import argparse
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from inputs import get_config, rhs_normal  # noqa: E402


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C3")
    ap.add_argument("--modes", default="1,all")
    args = ap.parse_args()
    from threadpoolctl import threadpool_limits
    cfg = get_config(args.config)
    dim = 3 if cfg.op == "stencil3d" else 2
    A = O.stencil_matrix(dim, cfg.m, cfg.beta)
    f = rhs_normal(cfg.n, cfg.seed)
    cores = len(os.sched_getaffinity(0))
    out = {"config": cfg.name, "n": cfg.n, "d": cfg.d, "k": cfg.k, "s": cfg.s, "zeta": cfg.zeta,
           "cpu_model": cpu_model(), "host_cores": cores, "what": "oracle.sgmres_cycle, cycle 0, full d (no early "
           "exit), x0 = 0", "runs": []}
    for mode in args.modes.split(","):
        lim = 1 if mode == "1" else cores
        with threadpool_limits(limits=lim):
            t0 = time.perf_counter()
            r = O.sgmres_cycle(lambda v: A @ v, f, np.zeros(cfg.n), cfg.d, cfg.k, cfg.s, cfg.zeta, cfg.seed, 0,
                               early_exit_factor=0.0)
            t = time.perf_counter() - t0
        rel = float(np.linalg.norm(f - A @ r["x"]) / np.linalg.norm(f))
        out["runs"].append({"threads": lim, "seconds": t, "columns": int(r["j"]), "rel_res_after_cycle": rel})
        print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
