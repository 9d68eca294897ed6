"""Oracle reference values at the FULL BASELINE config sizes -> tests/golden/oracle_<cfg>.json.

Calls ONLY ``oracle/`` (the plain fp64 CPU implementation of Alg. 1 / Alg. 2) and ``inputs/``
(seeded generators, no method arithmetic); nothing here touches the CUDA path.  The GPU tests
(tests/test_gpu_fullsize.py) compare the library's full-size runs against these files:

  sGMRES (C1-C4; Alg. 1, iterative form P:1351-1385, restarts P:938-957):
    cycles, columns (used, per cycle), per-cycle true residual hist_true, the r_est_j/||f||
    history of every cycle (hist_est), final relative residual, kappa(T) of the last cycle,
    flags, x at 64 seeded sample rows and ||x||_2.
  sRR (C5; Alg. 2, Eq. Mhat-form, Eq. srr-resid-est):
    the top nev+2 Ritz values in the canonical order of reading O23 (|theta| descending, ties by
    Im theta descending), their sketched residual estimates and true residuals, kappa(SB).

Usage:  python tools/make_oracle_golden.py C2 C3 ...   (default: all five)
Each file records the sha256 of the source text of the oracle/ and inputs/ functions it was produced by
(source_hash); the tests refuse a golden whose hash no longer matches (the oracle changed => regenerate).
Wall time on 8 host cores (numpy/scipy): C1 <1 s, C2 ~2 min, C3 ~10 min, C4 ~3 min, C5 ~5 min;
peak memory ~21 GB (C3/C5: B and AB at d = 300).
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
from inputs import get_config, rhs_normal, start_vector, start_block, random_csr_c4  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
NSAMPLE = 64


def _deps(method):
    """The oracle / inputs functions a golden of `method` depends on (its call graph)."""
    import inputs as I
    import oracle.sketch as OS
    common = [O.stencil_coeffs, O.toeplitz_1d, O.stencil_matrix, O.csr_matrix, OS.fmix64, OS.sketch_key, OS.floyd,
              OS.sketch_table, OS.sketch_matrix, O.thin_qr, I.rhs_normal, I.start_vector, I.random_csr_c4]
    if method == "sgmres":
        return common + [O.partial_arnoldi, O.sgmres_cycle, O.sgmres_solve]
    if method == "srr":
        return common + [O.partial_arnoldi, O.srr_eigs, O.srr_from_basis, O.select_ritz, O.srr.stabilized_pencil]
    return common + [O.spectral_box, O.block_chebyshev_basis, O.srr_eigs_block, O.srr_from_basis, O.select_ritz,
                     O.srr.stabilized_pencil, I.start_block]


def source_hash(method="sgmres"):
    """sha256 of the source text of every oracle/inputs function a golden of `method` is computed by (so adding
    unrelated functions to oracle/ does not invalidate it, and any change of those functions does)."""
    import inspect
    h = hashlib.sha256()
    for f in _deps(method):
        h.update(f.__module__.encode() + b"." + f.__qualname__.encode())
        h.update(inspect.getsource(f).encode())
    return h.hexdigest()


def sample_rows(n):
    """Seeded sample of rows at which x is recorded (shared by the GPU test)."""
    return np.sort(np.random.default_rng(12345).choice(n, size=min(NSAMPLE, n), replace=False))


def operator(cfg):
    if cfg.op == "csr":
        rp, ci, v, f = random_csr_c4(cfg.n, seed=cfg.seed)
        return O.csr_matrix(rp, ci, v, cfg.n), f
    dim = 3 if cfg.op == "stencil3d" else 2
    return O.stencil_matrix(dim, cfg.m, cfg.beta), None


def run_sgmres(cfg):
    A, f = operator(cfg)
    if f is None:
        f = rhs_normal(cfg.n, cfg.seed)
    t0 = time.time()
    # keep the per-cycle column counts: sgmres_solve concatenates hist_est, so run its cycles
    # through the same function with a wrapper that records out["j"] per cycle
    cols = []
    orig = O.sgmres.sgmres_cycle

    def rec(*a, **kw):
        out = orig(*a, **kw)
        cols.append(int(out["j"]))
        return out

    O.sgmres.sgmres_cycle = rec
    try:
        res = O.sgmres_solve(lambda v: A @ v, f, cfg.d, cfg.k, cfg.s, cfg.zeta, cfg.seed, tol=cfg.tol,
                             max_cycles=cfg.max_cycles, early_exit_factor=cfg.early_exit_factor)
    finally:
        O.sgmres.sgmres_cycle = orig
    wall = time.time() - t0
    x = res["x"]
    idx = sample_rows(cfg.n)
    return dict(
        config=cfg.name, method="sgmres", n=cfg.n, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed,
        tol=cfg.tol, max_cycles=cfg.max_cycles, early_exit_factor=cfg.early_exit_factor,
        cycles=int(res["cycles"]), columns=int(res["columns"]), columns_per_cycle=cols,
        rel_res_true=float(res["rel_res_true"]), hist_true=[float(v) for v in res["hist_true"]],
        hist_est=[float(v) for v in res["hist_est"]], cond_T=float(res["cond_T"]), flags=int(res["flags"]),
        x_norm=float(np.linalg.norm(x)), x_sample_rows=[int(i) for i in idx],
        x_sample=[float(v) for v in x[idx]], oracle_wall_s=wall)


def run_srr(cfg):
    A, _ = operator(cfg)
    v0 = start_vector(cfg.n, cfg.seed)
    nev = cfg.nev + 2
    t0 = time.time()
    out = O.srr_eigs(lambda v: A @ v, v0, cfg.d, cfg.k, cfg.s, cfg.zeta, cfg.seed, nev)
    wall = time.time() - t0
    th = out["theta"]
    return dict(
        config=cfg.name, method="srr", n=cfg.n, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed,
        nev=cfg.nev, nev_golden=len(th), theta_re=[float(t.real) for t in th], theta_im=[float(t.imag) for t in th],
        res_est=[float(v) for v in out["res_est"]], res_true=[float(v) for v in out["res_true"]],
        cond_SB=float(out["cond_SB"]), d_eff=int(out["basis"]["d_eff"]), oracle_wall_s=wall)


def run_srr_block(cfg):
    """C5B: block Chebyshev sRR -- oracle.srr_eigs_block with the closed-form
    spectral box of the stencil (oracle.spectral_box)."""
    A, _ = operator(cfg)
    Om = start_block(cfg.n, cfg.block, cfg.seed)
    dim = 3 if cfg.op == "stencil3d" else 2
    box = O.spectral_box(dim, cfg.m, cfg.beta)
    nev = cfg.nev + 2
    t0 = time.time()
    out = O.srr_eigs_block(lambda v: A @ v, Om, cfg.d // cfg.block, *box, cfg.s, cfg.zeta, cfg.seed, nev)
    wall = time.time() - t0
    th = out["theta"]
    return dict(
        config=cfg.name, method="srr_block", n=cfg.n, d=cfg.d, block=cfg.block, s=cfg.s, zeta=cfg.zeta,
        seed=cfg.seed, nev=cfg.nev, nev_golden=len(th), box=[float(v) for v in box],
        theta_re=[float(t.real) for t in th], theta_im=[float(t.imag) for t in th],
        res_est=[float(v) for v in out["res_est"]], res_true=[float(v) for v in out["res_true"]],
        cond_SB=float(out["cond_SB"]), oracle_wall_s=wall)


def main(names):
    for name in names:
        cfg = get_config(name)
        h = source_hash(cfg.method)
        print(f"[{name}] running the oracle at full size (n = {cfg.n}) ...", flush=True)
        g = {"sgmres": run_sgmres, "srr": run_srr, "srr_block": run_srr_block}[cfg.method](cfg)
        g["oracle_source_sha256"] = h
        g["produced_by"] = "tools/make_oracle_golden.py (oracle/ + inputs/ only)"
        g["host_cores"] = len(os.sched_getaffinity(0))
        path = os.path.join(GOLDEN, f"oracle_{name}.json")
        with open(path, "w") as fh:
            json.dump(g, fh, indent=1)
        print(f"[{name}] wrote {path} in {g['oracle_wall_s']:.1f} s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"])
