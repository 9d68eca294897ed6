"""The five BASELINE.json configurations (C1..C5), as plain metadata.

Readings of the config text are SURVEY.md section 8(c) O15-O21 and are repeated in
DESIGN.md section "Readings".  Nothing here computes anything of the method.
"""
from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class Config:
    name: str
    method: str            # "sgmres" | "srr"
    op: str                # "stencil2d" | "stencil3d" | "csr"
    m: int                 # grid points per side (stencil); 0 for CSR
    n: int                 # global dimension
    beta: float            # convection coefficient (stencil)
    seed: int              # seed of f / v0 / CSR and of the sketch hash
    d: int
    k: int
    s: int
    zeta: int = 8
    tol: float = 1e-8
    max_cycles: int = 1
    nev: int = 0
    block: int = 0         # block Krylov sRR: block size b (d = b p), 0 = single vector
    early_exit_factor: float = 0.25
    note: str = ""

    def with_(self, **kw):
        return replace(self, **kw)


CONFIGS = {
    # C1: 2D 32x32, no restarts (judged by parity only: 1e-8 unreachable)
    "C1": Config("C1", "sgmres", "stencil2d", 32, 32 * 32, 20.0, 0, 60, 2, 120,
                 max_cycles=1, note="single cycle, no restarts"),
    # C2: 2D 512x512, restarted until 1e-8, 1 GPU
    "C2": Config("C2", "sgmres", "stencil2d", 512, 512 * 512, 50.0, 1, 200, 4, 400,
                 max_cycles=50),
    # C3: 3D 160^3, restarted until 1e-8 (O15), 1/2/4/8 GPUs
    "C3": Config("C3", "sgmres", "stencil3d", 160, 160 ** 3, 30.0, 2, 300, 2, 600,
                 max_cycles=50),
    # C4: random CSR n=2M, 16 off-diagonal/row + diag 6, 1/2/4/8 GPUs
    "C4": Config("C4", "sgmres", "csr", 0, 2_000_000, 0.0, 3, 250, 2, 500,
                 max_cycles=50),
    # C5: sRR on 2D 2048x2048, 10 Ritz pairs of largest magnitude
    "C5": Config("C5", "srr", "stencil2d", 2048, 2048 * 2048, 10.0, 4, 300, 2, 600,
                 nev=10),
    # C5B (not a BASELINE config): C5's operator and small side (d = 300, s = 600, nev = 10) with
    # the block Chebyshev basis of P:1983-2008, b = 30 start vectors (Omega ~ N(0,1), seed 4), depth p = 10
    "C5B": Config("C5B", "srr_block", "stencil2d", 2048, 2048 * 2048, 10.0, 4, 300, 0, 600,
                  nev=10, block=30, note="block Chebyshev sRR, b = 30, p = 10"),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]
