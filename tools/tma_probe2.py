import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import paper_2111_00113_b200 as P
import oracle as O
from inputs import rhs_normal
dim, m, ncols, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
with P.Context(0) as ctx:
    A = P.StencilOperator(dim, m, 10.0)
    Ao = O.stencil_matrix(dim, m, 10.0)
    r0 = rhs_normal(m ** dim, 7)
    try:
        B, H = ctx.basis(A, r0, k=k, ncols=ncols)
        ref = O.partial_arnoldi(lambda v: Ao @ v, r0, ncols, k)
        print(dim, m, ncols, k, float(np.abs(B - ref["B"]).max()))
    except Exception as e:
        print(dim, m, ncols, k, "ERR", str(e)[:80])
