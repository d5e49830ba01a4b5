"""cpddg: B200-native (sm_100a, FP64) RAS/ORAS solve path for the closest point
method surface Helmholtz problem (arXiv:1909.08734), behind the reference's
operator / partition / solver interface.  See DESIGN.md."""
from .errors import ConfigError, CudaError, DivergenceError, InternalError, IoError  # noqa: F401

__all__ = ["api", "inputs", "errors"]
