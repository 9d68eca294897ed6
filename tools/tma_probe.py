"""Tiny probe of the TMA stencil path (first 8 basis columns vs the oracle)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402


def run():
    import paper_2111_00113_b200 as P
    import oracle as O
    from inputs import rhs_normal
    out = {}
    with P.Context(0) as ctx:
        for dim, m in [(2, 32), (3, 20)]:
            A = P.StencilOperator(dim, m, 10.0)
            Ao = O.stencil_matrix(dim, m, 10.0)
            r0 = rhs_normal(m ** dim, 7)
            try:
                B, H = ctx.basis(A, r0, k=2, ncols=8)
                ref = O.partial_arnoldi(lambda v: Ao @ v, r0, 8, 2)
                out[f"{dim}d"] = float(np.abs(B - ref["B"]).max())
            except Exception as e:
                out[f"{dim}d"] = str(e)
                break
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    run()
