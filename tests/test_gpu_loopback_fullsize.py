"""The library's OWN multi-rank code at the BASELINE scaling configurations, P = 8 ranks on one B200 through the
loopback transport (BASELINE configs 3 and 4 name 1/2/4/8 GPUs): C3 as 8 z-slabs of 20 planes with halo
exchange, pre-reduced partials and all-reduced partial sketches, and C4 as 8 contiguous row blocks with the gathered
remote x entries.  Each rank's solve must reproduce the ORACLE golden of the full problem (tests/golden/oracle_C*.json,
oracle-only): same cycles and used columns, per-cycle true residuals and every r_est at rtol 1e-4, the final residual
(recomputed with the oracle's operator) within the tolerance and within 2x of the oracle's; the replicated small side
gives bit-identical histories on every rank."""
import json
import os
import threading

import numpy as np
import pytest

import oracle as O
from inputs import get_config, partition_rows, rhs_normal, random_csr_c4

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
P = 8


def _run_ranks(fn):
    import paper_2111_00113_b200 as PK
    from paper_2111_00113_b200 import build
    build.build()
    grp = PK.LoopbackGroup(P)
    ctxs = [PK.Context(0, r, loopback=grp) for r in range(P)]
    out, err = [None] * P, [None] * P

    def work(r):
        try:
            out[r] = fn(ctxs[r], r)
        except Exception as e:  # pragma: no cover - reported below
            err[r] = e
    th = [threading.Thread(target=work, args=(r,), daemon=True) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in th), "a rank did not finish (collective mismatch?)"
    for c in ctxs:
        c.close()
    grp.close()
    for e in err:
        if e is not None:
            raise e
    return out


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_loopback_p8_full_size_vs_oracle_golden(name):
    import paper_2111_00113_b200 as PK
    cfg = get_config(name)
    with open(os.path.join(GOLDEN, f"oracle_{name}.json")) as fh:
        g = json.load(fh)
    n = cfg.n
    if cfg.op == "csr":
        rp, ci, v, f = random_csr_c4(n, seed=cfg.seed)
        Ao = O.csr_matrix(rp, ci, v, n)
        kind = "csr"
    else:
        f = rhs_normal(n, cfg.seed)
        Ao = O.stencil_matrix(3, cfg.m, cfg.beta)
        kind = "stencil3d"
    kw = dict(d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol, max_cycles=cfg.max_cycles,
              early_exit_factor=cfg.early_exit_factor)

    def fn(ctx, r):
        lo, hi = partition_rows(kind, n, cfg.m, P, r)
        if kind == "csr":
            rpl = (rp[lo:hi + 1] - rp[lo]).astype(np.int32)
            A = PK.CsrOperator(rpl, ci[rp[lo]:rp[hi]], v[rp[lo]:rp[hi]], n, lo, hi)
        else:
            A = PK.StencilOperator(3, cfg.m, cfg.beta, lo, hi)
        return ctx.sgmres_solve(A, f[lo:hi].copy(), **kw)

    outs = _run_ranks(fn)
    x = np.concatenate([o.x for o in outs])
    for o in outs:
        assert o.info["cycles"] == g["cycles"] and o.info["columns"] == g["columns"], o.info
        np.testing.assert_array_equal(o.hist, outs[0].hist)
    np.testing.assert_allclose(outs[0].hist_true, g["hist_true"], rtol=1e-4)
    np.testing.assert_allclose(outs[0].hist, g["hist_est"], rtol=1e-4)
    rel = np.linalg.norm(f - Ao @ x) / np.linalg.norm(f)
    assert rel <= cfg.tol, rel
    assert rel <= 2.0 * g["rel_res_true"] and g["rel_res_true"] <= 2.0 * rel, (rel, g["rel_res_true"])
