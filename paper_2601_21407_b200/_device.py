"""Device plumbing for the host shim: numpy <-> CUDA tensor moves, dtype codes,
the current CUDA stream handle.  PyTorch is used only for device memory and
streams; every computation runs in libhhb200.so.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as nat
from .errors import NativeLibraryError

_NP_TO_TORCH = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise NativeLibraryError("no CUDA device visible: the HH engine runs only on the GPU "
                                 "(there is no CPU fallback)")
    nat.load()
    return torch.device("cuda", torch.cuda.current_device())


def np_dtype(dtype) -> np.dtype:
    if isinstance(dtype, torch.dtype):
        return np.dtype({torch.float32: np.float32, torch.float64: np.float64}[dtype])
    d = np.dtype(dtype)
    if d not in _NP_TO_TORCH:
        raise NativeLibraryError(f"unsupported floating dtype {d}; use float32 or float64")
    return d


def torch_dtype(dtype) -> torch.dtype:
    return _NP_TO_TORCH[np_dtype(dtype)]


def code(dtype) -> int:
    return nat.F32 if np_dtype(dtype) == np.float32 else nat.F64


def is_dev(x) -> bool:
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_dev(x, dtype, dev=None) -> torch.Tensor:
    """Contiguous CUDA tensor of `dtype` holding x (no copy when already so)."""
    dev = dev or require_cuda()
    td = torch_dtype(dtype)
    if isinstance(x, torch.Tensor):
        t = x.to(device=dev, dtype=td)
    else:
        a = np.asarray(x, dtype=np_dtype(dtype))
        if not a.flags.c_contiguous:
            a = np.array(a, order="C")  # (np.ascontiguousarray would turn 0-d into 1-d)
        t = torch.from_numpy(a)
        t = t.to(dev, non_blocking=False)
    return t.contiguous()


def to_host(t: torch.Tensor, dtype=None) -> np.ndarray:
    """Device tensor -> numpy; a dtype change is done on the device first."""
    t = t.detach()
    if dtype is not None and np.dtype(dtype) in _NP_TO_TORCH and t.dtype != _NP_TO_TORCH[np.dtype(dtype)]:
        t = t.to(_NP_TO_TORCH[np.dtype(dtype)])
    a = t.cpu().numpy()
    return a if dtype is None else a.astype(dtype, copy=False)


def stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    return None if t is None else t.data_ptr()


INT64_MAX = 2 ** 63 - 1
