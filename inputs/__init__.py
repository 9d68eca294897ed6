"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no operator application, no
sketch, no Krylov recurrence, no least squares).  It only draws the random
inputs that BASELINE.json's configs name and packages the config metadata.
Both ``oracle/`` and the product path (``paper_2111_00113_b200``) may import it;
neither imports the other ("Independence").
"""
from .configs import CONFIGS, Config, get_config  # noqa: F401
from .generators import (  # noqa: F401
    rhs_normal,
    start_vector,
    start_block,
    random_csr_c4,
    partition_rows,
)
