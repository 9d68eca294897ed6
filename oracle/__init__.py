"""CPU fp64 ORACLE for sketched GMRES / sketched Rayleigh-Ritz (arXiv 2111.00113).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import or call
anything in this package.  The product path (``paper_2111_00113_b200``) never
imports it and shares no code with it: the two are independent implementations
written from PAPER.md.  Shared inputs come only from the ``inputs`` package,
which holds no method arithmetic.

Written plainly in numpy/scipy fp64 (paper precision, "IEEE double"), each
function citing the PAPER.md passage it follows (``P:<line>``).  Library
primitives used as single steps: sparse matrix-vector product (scipy.sparse),
thin QR (LAPACK dgeqrf via numpy), triangular solve, dense nonsymmetric
eigendecomposition (LAPACK dgeev via numpy).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to facts the
paper or mathematics fixes; see DESIGN.md "Oracle pins".  Functions with no pin:
none ("parity unpinned" would be stated here and in DESIGN.md).
"""
from .operators import (  # noqa: F401
    stencil_coeffs, stencil_matrix, csr_matrix, closed_form_eigs_1d,
    closed_form_eigs, toeplitz_1d, spectral_box,
)
from .sketch import (  # noqa: F401
    sketch_key, sketch_table, sketch_matrix, sketch_apply, fmix64,
    srft_key, srft_signs, srft_rows, srft_apply, SRFT,
)
from .krylov import partial_arnoldi, full_arnoldi, chebyshev_basis, block_chebyshev_basis  # noqa: F401
from .sgmres import (  # noqa: F401
    thin_qr, sgmres_cycle, sgmres_solve, gmres_exact_ls, whitened_basis, WARN_COND, WARN_BREAKDOWN, INFO_ADAPTIVE,
    INFO_WHITEN,
)
from .srr import srr_eigs, select_ritz, srr_from_basis, srr_eigs_block  # noqa: F401
