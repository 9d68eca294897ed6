#!/usr/bin/env python3
"""Benchmark: sGMRES time-to-1e-8 on BASELINE config C3 (3D convection-diffusion 160^3,
d=300, k=2, s=600, zeta=8), one process per GPU, plus the basis+sketch HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C3] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...

One "step" = one complete sGMRES solve to ||f - A x||/||f|| <= 1e-8 (all hot-path rows:
inputs resident -> residual -> truncated-Arnoldi basis -> sketch -> sketched QR/LS ->
assembly -> restart) with inputs already in HBM.  Multi-GPU: the z-slab row partition of
the same problem (strong scaling), NCCL halo + allreduce inside libsks.
Prints ONE JSON line on rank 0.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from inputs import get_config, rhs_normal, partition_rows  # noqa: E402

REASON_BITS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    def __init__(self, gpu_index):
        self.proc = None
        self.idx = gpu_index
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def __enter__(self):
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        try:
            rows = [l.strip().split(",") for l in open(self.path) if l.strip()]
            sm = [float(r[0]) for r in rows]
            mx = [float(r[1]) for r in rows]
            reasons = 0
            for r in rows:
                try:
                    reasons |= int(r[2].strip(), 16)
                except Exception:
                    pass
            names = [v for k, v in REASON_BITS.items() if reasons & k and v != "gpu_idle"]
            return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                    "reasons": names, "samples": len(sm)}
        except Exception as e:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "error": str(e)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return ws, rank, local


class OracleSampler:
    """The CPU oracle (oracle/, as it stands, never tuned) timed on BOUNDED samples of the bench workload at its
    real sizes (C3: n = 4,096,000, d = 300, s = 600), one component at a time; the cost of one restart cycle of
    oracle.sgmres_cycle is the sum of the components and the solve is `cycles` of them (the oracle always builds
    all d columns of a cycle; its cycle count at this config is tests/golden/oracle_C3.json's, 3):

      S       sketch_matrix(n, s, zeta, seed, c)                       (once per cycle)
      basis   partial_arnoldi at the real d (its n x d arrays, strided column access), stopped after 8 matvecs:
              per column = median interval between successive matvec calls 3..8 (one Arnoldi column: window
              dots, update, norm, strided stores, SpMV); first cost = time to the 2nd call (allocation and page
              faults of B and AB) minus one column
      SM      S @ AB on 32 of the d columns (scipy CSR x dense), x d/32
      rest    thin_qr + LS of an s x d problem, B y on 32 columns x d/32, the true-residual SpMV

    The BLAS pool is left at its default (all host cores); scipy's sparse products are single-threaded.
    tools/time_oracle_cycle.py measures one FULL cycle (1 thread and all cores) to check this sum
    (profiles/r02/oracle_cycle_c3.json)."""

    COMPONENTS = ("S", "basis", "SM", "rest")

    def __init__(self, cfg):
        import oracle as O
        self.O, self.cfg = O, cfg
        dim = 3 if cfg.op == "stencil3d" else 2
        self.A = O.stencil_matrix(dim, cfg.m, cfg.beta)
        self.f = rhs_normal(cfg.n, cfg.seed)
        self.t = {}
        self.cores = len(os.sched_getaffinity(0))
        self.cycles = 3
        gp = os.path.join(ROOT, "tests", "golden", f"oracle_{cfg.name}.json")
        if os.path.exists(gp):
            self.cycles = int(json.load(open(gp))["cycles"])
        self._S = None

    def _basis(self, nmv):
        class Stop(Exception):
            pass
        stamps = []
        A = self.A

        def mv(v):
            stamps.append(time.perf_counter())
            if len(stamps) > nmv:
                raise Stop
            return A @ v
        t0 = time.perf_counter()
        try:
            self.O.partial_arnoldi(mv, self.f, self.cfg.d, self.cfg.k)
        except Stop:
            pass
        iv = np.diff(stamps[1:])                      # calls 2..nmv+1: one Arnoldi column each
        per_col = float(np.median(iv))
        self.per_col = per_col
        self.first = max(stamps[1] - t0 - per_col, 0.0)

    def measure(self, comp):
        cfg, O = self.cfg, self.O
        t0 = time.perf_counter()
        if comp == "S":
            self._S = O.sketch_matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed, 0)
        elif comp == "basis":
            self._basis(8)
        else:
            S = self._S if self._S is not None else O.sketch_matrix(cfg.n, cfg.s, cfg.zeta, cfg.seed, 0)
            self._S = S
            M = np.ones((cfg.n, 32))
            t0 = time.perf_counter()
            if comp == "SM":
                S @ M
            else:
                C = np.random.default_rng(0).standard_normal((cfg.s, cfg.d))
                U, T = O.thin_qr(C)
                np.linalg.solve(T, U.T @ C[:, 0])
                M @ np.ones(32)
                x = np.zeros(cfg.n)
                np.linalg.norm(self.f - self.A @ x)
        dt = time.perf_counter() - t0
        self.t[comp] = dt
        return dt

    def estimate(self):
        t, d = self.t, self.cfg.d
        per_col, first = self.per_col, self.first
        cycle = t["S"] + first + per_col * d + t["SM"] * d / 32 + t["rest"] * d / 32
        return self.cycles * cycle, cycle, per_col

    def text(self):
        tot, cyc, pc = self.estimate()
        ms = ", ".join(f"{k} {v:.2f}s" for k, v in self.t.items())
        ms += f"; basis first cost {self.first:.2f}s"
        return (f"oracle (numpy/scipy, BLAS on {self.cores} host cores, sparse products 1 thread) on {self.cfg.name} "
                f"full n={self.cfg.n}, d={self.cfg.d}, s={self.cfg.s}: measured components [{ms}] -> "
                f"{pc:.3f} s per basis column, {cyc:.1f} s per cycle x {self.cycles} cycles (oracle golden) = "
                f"{tot:.1f} s per solve (extrapolated from the bounded samples; see bench.py OracleSampler)")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C3")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-oracle", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    ws, rank, local = dist_env()
    cfg = get_config(args.config)
    assert cfg.method == "sgmres"
    hbm_peak, peak_kind = peaks()
    metric = "sGMRES time-to-1e-8"
    workload = (f"{cfg.name}: {'3D 7-point' if cfg.op == 'stencil3d' else '2D 5-point'} convection-diffusion "
                f"m={cfg.m} (n={cfg.n}), beta={cfg.beta}, f~N(0,1) seed {cfg.seed}; sGMRES d={cfg.d} k={cfg.k} "
                f"s={cfg.s} zeta={cfg.zeta}, restarted to 1e-8")

    if args.impl == "reference":
        if rank != 0:
            return 0
        # the oracle as it stands, on the host cores: each step times ONE bounded component of the workload
        # (OracleSampler), the warm-up covers all of them; every timed step reports the full-solve estimate
        # from the latest measurement of each component
        smp = OracleSampler(cfg)
        comps = OracleSampler.COMPONENTS
        for i in range(max(args.warmup, len(comps))):
            smp.measure(comps[i % len(comps)])
        vals, walls = [], []
        for i in range(args.steps):
            walls.append(smp.measure(comps[i % len(comps)]))
            vals.append(smp.estimate()[0])
        v = statistics.mean(vals)
        wall = statistics.mean(walls)
        line = {"impl": "reference", "metric": metric, "value": v, "unit": "s", "n_gpus": args.gpus,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": wall * 1e3, "higher_is_better": False,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload, "parallelism": "cpu-oracle",
                           "step": "one bounded oracle component per step (ms_per_step = its measured wall "
                                   "time); value = the full-solve estimate from all components"},
                "cpu_baseline": {"value": v, "unit": "s", "cores": smp.cores, "kind": "oracle",
                                 "sample": smp.text()},
                "e2e": {"value": v, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return 0

    import torch
    import paper_2111_00113_b200 as P
    from paper_2111_00113_b200 import build as B
    B.build()
    dev = local if torch.cuda.device_count() > 1 else 0
    torch.cuda.set_device(dev)
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        idt = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(P.get_unique_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        nccl_id = bytes(idt.cpu().tolist())
    ctx = P.Context(dev, rank, ws, nccl_id)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream)
    rb, re_ = partition_rows(cfg.op, cfg.n, cfg.m, ws, rank)
    dim = 3 if cfg.op == "stencil3d" else 2
    A = P.StencilOperator(dim, cfg.m, cfg.beta, rb, re_)
    f_full = rhs_normal(cfg.n, cfg.seed)
    f_host = torch.from_numpy(f_full[rb:re_].copy()).pin_memory()
    f_dev = f_host.cuda()
    kw = dict(d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol, max_cycles=cfg.max_cycles,
              early_exit_factor=cfg.early_exit_factor, time_steps=True, time_stride=16)

    def barrier():
        torch.cuda.synchronize()
        if ws > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        res = ctx.sgmres_solve(A, f_dev, **kw)
    barrier()
    infos = []
    with ClockSampler(dev) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for _ in range(args.steps):
            res = ctx.sgmres_solve(A, f_dev, **kw)
            infos.append(res.info)
        ev1.record(stream)
        barrier()
    t_dev = ev0.elapsed_time(ev1) * 1e-3 / args.steps
    # end-to-end: host (pinned) buffers through the C-ABI, copies inside the timed region
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    x_host = torch.zeros_like(f_host).pin_memory()
    e0.record(stream)
    for _ in range(max(1, args.steps // 2)):
        r2 = ctx.sgmres_solve(A, f_host, out=x_host, **kw)  # x0 = 0; f pinned in, x pinned out
    e1.record(stream)
    barrier()
    t_e2e = e0.elapsed_time(e1) * 1e-3 / max(1, args.steps // 2)

    # roofline of the dominant kernel (the fused Arnoldi step): algorithmic bytes of its launches
    # / their summed duration, both from the library: CUDA events on the main stream inside the timed
    # solves (SKS_OPT_TIME_STEPS) around windows of time_stride = 16 consecutive step launches within a
    # sketch batch, so consecutive launches keep their programmatic (PDL) overlap as in the untimed
    # pipeline; SKS_TIME_WINDOW=1 brackets single launches instead (each then loses that overlap)
    t_basis = statistics.mean(i["t_basis_s"] for i in infos)
    bytes_basis = statistics.mean(i["bytes_basis"] for i in infos)
    steps_per_solve = statistics.mean(i["steps"] for i in infos)
    launches = sum(i["kernel_launches"] for i in infos)
    t_step = sum(i["t_step_s"] for i in infos)
    n_step = sum(i["steps_timed"] for i in infos)
    b_step = sum(i["bytes_step"] for i in infos)
    step_gbs = b_step / t_step / 1e9 if t_step > 0 else 0.0
    gbs = bytes_basis / t_basis / 1e9 if t_basis > 0 else 0.0
    vals = torch.tensor([t_dev, t_e2e, gbs, t_basis, step_gbs], dtype=torch.float64, device="cuda")
    if ws > 1:
        mx = vals.clone()
        torch.distributed.all_reduce(mx, op=torch.distributed.ReduceOp.MAX)
        sm = vals.clone()
        torch.distributed.all_reduce(sm, op=torch.distributed.ReduceOp.SUM)
        t_dev, t_e2e, t_basis = float(mx[0]), float(mx[1]), float(mx[3])
        gbs, step_gbs = float(sm[2]), float(sm[4])  # aggregate algorithmic GB/s over all GPUs
    clocks = clk.summary()
    info = infos[-1]
    # check the answer (true residual recomputed by the library is in info)
    ok = info["rel_res_true"] <= cfg.tol
    if rank == 0:
        cpu = None
        if not args.no_oracle and ws == 1:  # the CPU baseline is taken at N = 1 only
            try:
                smp = OracleSampler(cfg)
                for comp in OracleSampler.COMPONENTS:
                    smp.measure(comp)
                v = smp.estimate()[0]
                cpu = {"value": v, "unit": "s", "cores": smp.cores, "kind": "oracle", "sample": smp.text()}
                cp = os.path.join(ROOT, "profiles", "r02", "oracle_cycle_c3.json")
                if cfg.name == "C3" and os.path.exists(cp):
                    mc = json.load(open(cp))
                    cpu["measured_full_cycle"] = {
                        "runs": mc["runs"], "cpu_model": mc["cpu_model"], "host_cores": mc["host_cores"],
                        "x_cycles_estimate_s": [r["seconds"] * smp.cycles for r in mc["runs"]],
                        "source": "profiles/r02/oracle_cycle_c3.json (tools/time_oracle_cycle.py on the GPU box)"}
            except Exception as e:  # pragma: no cover
                cpu = {"value": None, "unit": "s", "cores": 0, "kind": "oracle", "sample": f"failed: {e}"}
        traffic = None
        tp = os.path.join(ROOT, "profiles", "step_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(cfg.name)
            except Exception:
                traffic = None
        peak_total = hbm_peak * ws
        line = {
            "metric": metric, "value": t_dev, "unit": "s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev * 1e3, "higher_is_better": False, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload, "n": cfg.n, "d": cfg.d, "k": cfg.k, "s": cfg.s, "zeta": cfg.zeta,
                       "tol": cfg.tol, "parallelism": f"rows1d-{ws}",
                       "l2": "no flush: per-step working set (basis 9.9 GB) >> 126 MB L2",
                       "cycles": info["cycles"], "columns": info["columns"],
                       "columns_generated": info["columns_generated"], "rel_res_true": info["rel_res_true"],
                       "converged": bool(ok)},
            "basis_sketch": {"columns_per_s": steps_per_solve / t_basis if t_basis > 0 else None,
                             "gbs": gbs, "t_basis_s": t_basis, "t_solve_s": t_dev,
                             "frac_of_hbm": gbs / peak_total},
            "roofline": {"bound": "hbm", "kernel": "step3d_zmp_kernel (fused truncated-Arnoldi step)",
                         "achieved": step_gbs, "peak": peak_total, "unit": "GB/s", "frac": step_gbs / peak_total,
                         "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json hbm_gbs, copy burst)", "traffic": traffic,
                         "bytes_per_launch_alg": b_step / max(n_step, 1),
                         "avg_launch_us": t_step / max(n_step, 1) * 1e6, "launches_timed": int(n_step),
                         # sampled launches (every 16th) -> mean duration x step launches per solve
                         "share_of_solve": (t_step / max(n_step, 1)) * steps_per_solve / t_dev
                         if t_dev > 0 else None},
            "cpu_baseline": cpu,
            "e2e": {"value": t_e2e, "unit": "s", "h2d_bytes_per_step": int(8 * (re_ - rb)),
                    "d2h_bytes_per_step": int(8 * (re_ - rb))},
            "gpu_launches": int(launches),
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
