"""Probe: time the plain y = A x stencil kernel at C3 size (for roofline comparisons)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2111_00113_b200 as P
ctx = P.Context(0)
m = 160
x = torch.randn(m ** 3, dtype=torch.float64, device="cuda")
A = P.StencilOperator(3, m, 30.0)
for _ in range(5):
    y = ctx.apply_operator(A, x)
torch.cuda.synchronize()
print("ok")
