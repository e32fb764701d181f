"""B200-native Hodgkin-Huxley hot path of BrainFuse (arXiv 2601.21407).

Drop-in for the reference package's `hhengine.dynamics`, `hhengine.adjoint`,
`hhengine.defaults` and `hhengine.errors` modules; all compute runs in the
sm_100a library libhhb200.so (include/hhb200.h) -- there is no CPU path.
"""

from . import errors
from .errors import (ConfigurationError, GradientOverflowError, HHEngineError,
                     NativeLibraryError, NumericalOverflowError, TrainingDivergedError, UsageError)

__all__ = ["errors", "ConfigurationError", "GradientOverflowError", "HHEngineError",
           "NativeLibraryError", "NumericalOverflowError", "TrainingDivergedError", "UsageError"]
__version__ = "0.1.0"
