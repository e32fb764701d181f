"""Exception contract of the drop-in API.

Same class names, hierarchy and `step_index` / `epoch` attributes as the
reference (`hhengine/errors.py:4-51`), so callers that catch the reference's
exceptions keep working.  The GPU path raises them from the host shim after
reading the device-side first-bad-step word (see dynamics.simulate).
"""

from __future__ import annotations


class HHEngineError(Exception):
    """Root of every error the engine raises (errors.py:4)."""


class ConfigurationError(HHEngineError):
    """Bad parameter set or a gate-layout mismatch (errors.py:8)."""


class UsageError(HHEngineError):
    """Structurally invalid call arguments (errors.py:12)."""


class _StepIndexed(HHEngineError):
    def __init__(self, message: str, step_index: int | None = None):
        self.step_index = step_index
        if step_index is not None:
            message = f"{message} (step {step_index})"
        super().__init__(message)


class NumericalOverflowError(_StepIndexed):
    """Membrane potential became non-finite in the forward pass (errors.py:16-24)."""


class GradientOverflowError(_StepIndexed):
    """Adjoint state became non-finite in the backward pass (errors.py:27-35)."""


class TrainingDivergedError(HHEngineError):
    """Training loss became non-finite (errors.py:38-43)."""

    def __init__(self, message: str, epoch: int | None = None):
        self.epoch = epoch
        if epoch is not None:
            message = f"{message} (epoch {epoch})"
        super().__init__(message)


class KeygenError(HHEngineError):
    """Kept for API completeness (errors.py:46); the cipher is out of scope."""


class KeyIntegrityError(HHEngineError):
    """Kept for API completeness (errors.py:50); the cipher is out of scope."""


class NativeLibraryError(HHEngineError):
    """The CUDA library is missing, failed to load, or returned an error code.

    Not in the reference: the reference has no native code.  There is no CPU
    fallback, so a missing library is always fatal.
    """


class ExchangeError(HHEngineError):
    """The multi-GPU spike exchange failed: an NCCL asynchronous error, or a
    step that did not complete within the exchange timeout (the communicator
    is aborted first, so no rank stays blocked in the collective).  Not part
    of the reference's error contract (the reference is single-process)."""
