"""B200-native Riemannian geodesic ray tracer (drop-in for the rray render path).

The compute path is the CUDA library ``csrc/librray_cuda.so`` (sm_100a) behind
the C-ABI of ``include/rray_cuda.h``; ``render`` wraps it with the reference's
API names.  Importing the package does not load the library; the first
``Renderer`` does, and fails loudly when it is missing.
"""
from .errors import (ConfigError, DegenerateBasis, DeviceError, Error, IoError,  # noqa: F401
                     NumericError, ParseError, SingularJacobian, SingularMatrix,
                     ValidationError)
from .config import load_config, parse_config, serialize_config  # noqa: F401

__all__ = ["load_config", "parse_config", "serialize_config"]
