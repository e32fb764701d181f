"""B200-native Hodgkin-Huxley hot path of BrainFuse (arXiv 2601.21407).

Drop-in for the reference package `hhengine`: the same-named modules
(`dynamics`, `adjoint`, `defaults`, `errors`, `learn`, `cortex`, `connectivity`,
`morphology`, `reference`) expose every public name of the reference's; plus
`layer` (the tcgen05 + HH autograd layer), `network` (the device cortex) and
`population`.  All compute runs in the sm_100a library libhhb200.so
(include/hhb200.h) -- there is no CPU path.
"""

from . import errors
from .errors import (ConfigurationError, GradientOverflowError, HHEngineError,
                     NativeLibraryError, NumericalOverflowError, TrainingDivergedError, UsageError)

__all__ = ["errors", "ConfigurationError", "GradientOverflowError", "HHEngineError",
           "NativeLibraryError", "NumericalOverflowError", "TrainingDivergedError", "UsageError"]
__version__ = "0.1.0"
