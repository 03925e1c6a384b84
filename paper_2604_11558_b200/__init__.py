"""B200-native split exponential Euler engine (arXiv 2604.11558 hot path).

Drop-in for the time-stepping path of the reference package ``curvipat``:
host-side setup (operators, phi1 tables) in NumPy/SciPy, every per-step
operation in hand-written sm_100a CUDA (libcurvigpu.so, C ABI in
include/curvigpu.h) called through ctypes on PyTorch-owned device memory.
"""

from . import configs, coupled, ensemble, integrators, models, operators, phifun  # noqa: F401
from ._native import LIB_PATH, EngineError  # noqa: F401

__version__ = "0.1.0"
