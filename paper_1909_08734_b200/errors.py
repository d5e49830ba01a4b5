"""Exception hierarchy mirroring the reference (proj/include/cpdd/core.hpp:73-95).

The C ABI returns status codes (include/cpddg.h); these classes restore the
reference's exception types on the Python side so callers keep the same
error behaviour (and exit codes 2/3/4/1, proj/tools/cpm.cpp:181-193).
"""
from ._lib import CpddgError


class ConfigError(CpddgError):
    """Invalid or out-of-range configuration (exit code 2)."""


class IoError(CpddgError):
    """File-system problem (exit code 4)."""


class DivergenceError(CpddgError):
    """Iteration diverged, residual non-finite, or a singular local factor (exit code 3)."""


class InternalError(CpddgError):
    """Violated internal invariant (exit code 1)."""


class CudaError(CpddgError):
    """CUDA runtime failure on the device path."""
