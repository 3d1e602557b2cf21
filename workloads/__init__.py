"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This package holds ONLY input generation (supports, coefficients, liftings,
points).  It contains none of the method's arithmetic (no evaluation, no
derivatives, no solves), so both `oracle/` and `paper_2111_14317_b200/` may
consume its output without sharing any computation (task rule ③).
"""
from .systems import (  # noqa: F401
    System, cyclic, katsura, noon, chandra, random_dense, diagonal, from_terms,
    MASTER_SEED,
)
from .points import random_points, random_log_points, random_extended_points  # noqa: F401
