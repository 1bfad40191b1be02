"""B200-native hot path of arXiv 1808.02937 (H-matrix preconditioned SEM solve of
the 1-D two-sided Riemann-Liouville fractional diffusion equation).

The compute lives in libfde.so (CUDA, sm_100a; C-ABI in include/fde.h);
`fde` is the ctypes binding.
"""
from . import fde  # noqa: F401
from .fde import *  # noqa: F401,F403
