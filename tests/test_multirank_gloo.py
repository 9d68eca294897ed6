"""Multi-rank host logic on CPU (world size 2, gloo), no GPU.

The B200 path shards rows of A, B and the vectors in contiguous blocks of whole lines/planes
(DESIGN.md section 8): per column a halo exchange of G = 2 ghost planes with the two
neighbour ranks and an allreduce of per-rank partial sums; per batch an allreduce of the
partial sketches.  These tests run the same protocol with torch.distributed (gloo) on numpy
data and check it against the single-process oracle:

  * the partition (inputs.partition_rows, mirrored by sks_partition) tiles [0, n) exactly,
    computed independently on every rank;
  * the NCCL unique id made by libsks on rank 0 reaches every rank unchanged;
  * sum over ranks of S_rows M_rows (each rank hashing only its global rows) == S M, i.e. the
    sketch allreduce reproduces the global sketch (S's column r depends on r only);
  * a stencil apply on each rank's slab, with G ghost planes filled by the neighbour
    exchange (send the first/last G owned planes to rank -/+ 1, zero at the physical
    boundary), equals the global operator's rows; the partial dot products allreduced over
    ranks equal the global ones;
  * bench.py's timing reduction takes the MAX over ranks.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
WS = 2
G = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _halo_exchange(vec, plane, nz, rank, ws):
    """vec: (nz + 2G) * plane ghost-layout slab; fills the ghost planes from the neighbours
    (the protocol of api.cu halo_exchange)."""
    cnt = G * plane
    lo, hi = rank - 1, rank + 1
    reqs = []
    if lo >= 0:
        reqs.append(dist.isend(torch.from_numpy(vec[G * plane:G * plane + cnt].copy()), lo))
        buf_lo = torch.empty(cnt, dtype=torch.float64)
        reqs.append(dist.irecv(buf_lo, lo))
    if hi < ws:
        reqs.append(dist.isend(torch.from_numpy(vec[nz * plane:nz * plane + cnt].copy()), hi))
        buf_hi = torch.empty(cnt, dtype=torch.float64)
        reqs.append(dist.irecv(buf_hi, hi))
    for r in reqs:
        r.wait()
    if lo >= 0:
        vec[:cnt] = buf_lo.numpy()
    if hi < ws:
        vec[(nz + G) * plane:(nz + 2 * G) * plane] = buf_hi.numpy()


def _slab_apply(vec, m, nz, dim, coeffs):
    """y = A x on the owned planes of a ghost-layout slab (x fastest, Dirichlet in x/y)."""
    cc, cmi, cpl = coeffs
    if dim == 3:
        x = vec.reshape(nz + 2 * G, m, m)
        own = x[G:G + nz]
        y = cc * own
        y = y + cmi * x[G - 1:G - 1 + nz] + cpl * x[G + 1:G + 1 + nz]
        y[:, 1:, :] += cmi * own[:, :-1, :]
        y[:, :-1, :] += cpl * own[:, 1:, :]
        y[:, :, 1:] += cmi * own[:, :, :-1]
        y[:, :, :-1] += cpl * own[:, :, 1:]
    else:
        x = vec.reshape(nz + 2 * G, m)
        own = x[G:G + nz]
        y = cc * own + cmi * x[G - 1:G - 1 + nz] + cpl * x[G + 1:G + 1 + nz]
        y[:, 1:] += cmi * own[:, :-1]
        y[:, :-1] += cpl * own[:, 1:]
    return y.reshape(-1)


def _worker(rank, port, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WS)
    import sys
    sys.path.insert(0, ROOT)
    import oracle as O
    from inputs import partition_rows, rhs_normal
    out = {}
    try:
        # ---- partition: independently computed blocks tile [0, n)
        for kind, n, m in [("stencil3d", 24 ** 3, 24), ("stencil2d", 50 * 50, 50), ("csr", 1001, 0)]:
            rb, re_ = partition_rows(kind, n, m, WS, rank)
            t = torch.tensor([rb, re_], dtype=torch.int64)
            allb = [torch.zeros(2, dtype=torch.int64) for _ in range(WS)]
            dist.all_gather(allb, t)
            blocks = [tuple(b.tolist()) for b in allb]
            ok = blocks[0][0] == 0 and blocks[-1][1] == n and all(blocks[i][1] == blocks[i + 1][0]
                                                                   for i in range(WS - 1))
            unit = {"stencil3d": m * m, "stencil2d": m, "csr": 1}[kind]
            ok = ok and all((b[0] % unit == 0 and b[1] % unit == 0) for b in blocks)
            out[f"partition_{kind}"] = bool(ok)
        # ---- unique id broadcast (bytes made by libsks on rank 0)
        idt = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            try:
                import paper_2111_00113_b200 as P
                idt = torch.frombuffer(bytearray(P.get_unique_id()), dtype=torch.uint8).clone()
            except Exception:
                idt = torch.arange(128, dtype=torch.uint8)
        dist.broadcast(idt, 0)
        h = torch.tensor([int(idt.to(torch.int64).sum()), int(idt[0]), int(idt[127])], dtype=torch.int64)
        hs = [torch.zeros(3, dtype=torch.int64) for _ in range(WS)]
        dist.all_gather(hs, h)
        out["uid_equal"] = all(torch.equal(hs[0], x) for x in hs)
        # ---- sketch allreduce == global sketch
        n, s, zeta, c = 3000, 64, 8, 5
        M = np.random.default_rng(11).standard_normal((n, c))
        rb, re_ = partition_rows("csr", n, 0, WS, rank)
        part = O.sketch_apply(M[rb:re_], s, zeta, seed=3, cycle=2, row_begin=rb, n=n)
        t = torch.from_numpy(np.ascontiguousarray(part))
        dist.all_reduce(t)
        full = O.sketch_apply(M, s, zeta, seed=3, cycle=2)
        out["sketch_err"] = float(np.linalg.norm(t.numpy() - full) / np.linalg.norm(full))
        # ---- halo exchange + slab stencil == global operator; partial dots allreduced
        for dim, m, beta in [(3, 12, 30.0), (2, 40, 20.0)]:
            n = m ** dim
            kind = "stencil3d" if dim == 3 else "stencil2d"
            plane = m * m if dim == 3 else m
            rb, re_ = partition_rows(kind, n, m, WS, rank)
            nz = (re_ - rb) // plane
            x = rhs_normal(n, 5)
            vec = np.zeros((nz + 2 * G) * plane)
            vec[G * plane:(G + nz) * plane] = x[rb:re_]
            _halo_exchange(vec, plane, nz, rank, WS)
            a, b, cc_ = O.stencil_coeffs(m, beta)
            coeffs = (dim * a, b, cc_)
            y = _slab_apply(vec, m, nz, dim, coeffs)
            yg = O.stencil_matrix(dim, m, beta) @ x
            out[f"halo_err_{dim}d"] = float(np.abs(y - yg[rb:re_]).max() / np.abs(yg).max())
            d2 = torch.tensor([float(y @ y), float(y @ x[rb:re_])], dtype=torch.float64)
            dist.all_reduce(d2)
            ref = np.array([yg @ yg, yg @ x])
            out[f"dots_err_{dim}d"] = float(np.abs(d2.numpy() - ref).max() / np.abs(ref).max())
        # ---- bench timing reduction: max over ranks
        tt = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        out["max_time"] = float(tt)
    finally:
        dist.destroy_process_group()
    results[rank] = out


@pytest.mark.timeout(300)
def test_multirank_protocol_gloo():
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    results = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, results)) for r in range(WS)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(240)
        assert p.exitcode == 0, f"rank exited with {p.exitcode}"
    for r in range(WS):
        o = results[r]
        for kind in ("stencil3d", "stencil2d", "csr"):
            assert o[f"partition_{kind}"], (r, kind)
        assert o["uid_equal"]
        assert o["sketch_err"] <= 1e-14, o["sketch_err"]
        for dim in (2, 3):
            assert o[f"halo_err_{dim}d"] <= 1e-14, o
            assert o[f"dots_err_{dim}d"] <= 1e-13, o
        assert o["max_time"] == float(WS)
