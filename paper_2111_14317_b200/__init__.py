"""B200-native hot path of arXiv 2111.14317 (GEMM-style evaluation of polyhedral homotopies
and consolidated Euler/Newton directions).  See DESIGN.md.

The CUDA library (lib/libpht.so) is required; importing this package without it raises.
"""
from ._lib import PhtError, load as _load_lib  # noqa: F401
from ._lib import (PT_OK, PT_ZERO_COORD, PT_NONFINITE, PT_SINGULAR, PT_STEP_UNDERFLOW,  # noqa: F401
                   PT_MAX_STEPS, PT_DIVERGED, PT_FLOOR, PHT_MAX_N)

_load_lib()

from .api import System, launch_count, specialize_compile, specialize_source  # noqa: E402,F401
