"""ctypes binding of the C-ABI library (include/hhb200.h).

This is the only place Python touches native code.  The library is loaded from
the package directory (built in-tree by `_build.py`); if it is missing or the
ABI version differs, every compute entry point raises NativeLibraryError --
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .errors import ConfigurationError, NativeLibraryError, UsageError

# HHB200_LIB: an alternative build of the library (kernel-variant experiments)
LIB_PATH = os.environ.get("HHB200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhhb200.so")
ABI_VERSION = 3
MAX_GATES = 8
MAX_CHANNELS = 8

F32, F64 = 0, 1
RATE_KIND = {"linoid": 0, "exp": 1, "sigmoid": 2}
SUR_KIND = {"sigmoid-derivative": 0, "rectangular": 1}

OK, EINVAL, ENOTSUP, ECUDA = 0, 22, 95, 1000


class Rate(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32),
                ("a", C.c_double), ("v0", C.c_double), ("b", C.c_double)]


class Gate(C.Structure):
    _fields_ = [("alpha", Rate), ("beta", Rate), ("exponent", C.c_int32), ("channel", C.c_int32)]


class Channel(C.Structure):
    _fields_ = [("g_max", C.c_double), ("e_rev", C.c_double),
                ("gate_begin", C.c_int32), ("gate_count", C.c_int32)]


class Params(C.Structure):
    _fields_ = [("n_gates", C.c_int32), ("n_channels", C.c_int32),
                ("c_m", C.c_double), ("dt", C.c_double), ("v_theta", C.c_double),
                ("v_rest", C.c_double), ("rate_scale", C.c_double),
                ("gates", Gate * MAX_GATES), ("channels", Channel * MAX_CHANNELS)]


class Thalamic(C.Structure):
    """hhb_thalamic_t"""
    _fields_ = [("offsets", C.c_void_p), ("weights", C.c_void_p), ("id_base", C.c_int64), ("t_on", C.c_int64),
                ("t_off", C.c_int64), ("threshold", C.c_uint32), ("reserved", C.c_uint32), ("seed", C.c_uint64)]


class Surrogate(C.Structure):
    _fields_ = [("kind", C.c_int32), ("reserved", C.c_int32), ("width", C.c_double)]


_vp, _i64, _i32, _dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double

# name -> (restype, argtypes); mirrors include/hhb200.h one to one
SIGNATURES = {
    "hhb_abi_version": (_i32, []),
    "hhb_last_error": (C.c_char_p, []),
    "hhb_check_params": (_i32, [C.POINTER(Params)]),
    "hhb_forward": (_i32, [C.POINTER(Params), _i32, _i64, _i64,
                           _vp, _vp, _i64, _vp, _vp,
                           _vp, _i64, _i64,
                           _vp, _i64,
                           _vp, _i64,
                           _vp, _i64, _i64,
                           _i64, _vp, _vp]),
    "hhb_forward_ex": (_i32, [C.POINTER(Params), _i32, _i64, _i64,
                              _vp, _vp, _i64, _vp, _vp,
                              _vp, _i64, _i64,
                              _vp, _i64,
                              _vp, _i64,
                              _vp, _i64,
                              _vp, _i64, _i64,
                              _i64, _vp, _vp, _vp, _vp]),
    "hhb_forward_ex2": (_i32, [C.POINTER(Params), _i32, _i64, _i64,
                               _vp, _vp, _i64, _vp, _vp,
                               _vp, _i64, _i64,
                               _vp, _i64,
                               _vp, _i64,
                               _vp, _i64,
                               _vp, _i64, _i64,
                               _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "hhb_forward_partials": (_i64, [_i64]),
    "hhb_backward": (_i32, [C.POINTER(Params), C.POINTER(Surrogate), _i32, _i64, _i64,
                            _vp, _i64, _i64,
                            _vp, _i64, _i64, _vp,
                            _vp, _i64, _vp, _i64,
                            _vp, _vp, _i64,
                            _vp, _i64,
                            _vp, _vp,
                            _i64, _vp, _vp]),
    "hhb_backward_ex": (_i32, [C.POINTER(Params), C.POINTER(Surrogate), _i32, _i64, _i64,
                               _vp, _i64, _i64,
                               _vp, _i64, _i64, _vp,
                               _vp, _i64, _vp, _i64,
                               _vp, _vp, _i64,
                               _vp, _i64,
                               _vp, _vp,
                               _i64, _vp,
                               _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp]),
    "hhb_forward_poisson": (_i32, [C.POINTER(Params), _i32, _i64, _i64,
                                   _vp, _vp, _i64, _vp, _vp,
                                   C.c_uint64, _i64, _dbl, _dbl,
                                   _vp, _i64,
                                   _vp, _i64,
                                   _vp, _i64, _i64,
                                   _i64, _vp, _vp]),
    "hhb_backward_partials": (_i64, [_i64, _i32]),
    "hhb_gate_rates": (_i32, [C.POINTER(Gate), _dbl, _i32, _i64, _vp, _vp, _vp, _vp]),
    "hhb_rate_eval": (_i32, [C.POINTER(Rate), _i32, _i32, _i64, _vp, _vp, _vp]),
    "hhb_gate_step": (_i32, [_i32, _i64, _vp, _vp, _vp, _dbl, _vp, _vp]),
    "hhb_ionic_current": (_i32, [C.POINTER(Params), _i32, _i64, _vp, _vp, _i64, _vp, _vp]),
    "hhb_spike_detect": (_i32, [_i32, _i64, _vp, _vp, _dbl, _vp, _vp]),
    "hhb_surrogate_grad": (_i32, [C.POINTER(Surrogate), _i32, _i64, _vp, _vp, _vp]),
    "hhb_unpack_spikes": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "hhb_unpack_spikes_f32": (_i32, [_vp, _i64, _i64, _i64, _vp, _i64, _vp]),
    "hhb_poisson_current": (_i32, [_i32, _i64, _i64, C.c_uint64, _i64, _i64, _dbl, _dbl,
                                   _vp, _i64, _vp]),
    "hhb_pipe_probe": (_i32, [_i32, _i64, _vp, C.POINTER(C.c_int64), _vp]),
    "hhb_gemm": (_i32, [_i32, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp]),
    "hhb_gemm_workspace": (_i64, [_i64, _i64, _i32]),
    "hhb_gemm_ex": (_i32, [_i32, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp]),
    "hhb_gemm_ex2": (_i32, [_i32, _i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _i64,
                             _vp]),
    "hhb_transpose": (_i32, [_i32, _i64, _i64, _vp, _i64, _vp, _i64, _vp]),
    "hhb_cast_bf16": (_i32, [_i64, _vp, _vp, _vp]),
    "hhb_split_rows_bf16": (_i32, [_i64, _i64, _vp, _i64, _vp, _i64, _vp]),
    "hhb_spk_exchange_available": (_i32, []),
    "hhb_spk_exchange_unique_id": (_i32, [_vp, _i64]),
    "hhb_spk_exchange_init": (_i32, [_vp, _i32, _i32, _i64, C.POINTER(_vp)]),
    "hhb_spk_exchange_allgather": (_i32, [_vp, _vp, _vp, _vp]),
    "hhb_spk_step": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp]),
    "hhb_spk_exchange_status": (_i32, [_vp]),
    "hhb_spk_exchange_abort": (_i32, [_vp]),
    "hhb_spk_exchange_destroy": (_i32, [_vp]),
    "hhb_split3_bf16": (_i32, [_i64, _i64, _vp, _i64, _vp, _i64, _i64, _i32, _vp]),
    "hhb_col_sum": (_i32, [_i64, _i64, _vp, _i64, _vp, _vp, _vp]),
    "hhb_col_sum_scratch": (_i64, [_i64, _i64]),
    "hhb_col_sum_ex": (_i32, [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp]),
    "hhb_gemm_f32a": (_i32, [_i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _vp, _vp, _i64, _i32, _vp, _vp, _i64,
                             _i64, _vp]),
    "hhb_gemm_f32b": (_i32, [_i64, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _i32, _vp, _i64, _i32, _vp, _vp]),
    "hhb_sum_f64": (_i32, [_i64, _vp, C.c_double, _vp, _vp, _vp]),
    "hhb_cortex_input": (_i32, [_i32, _i64, _i64, _i64, _vp, _vp, _dbl, _i32, _vp, _vp, _dbl, _dbl,
                                C.c_uint64, _i64, _vp, _vp, _dbl, _vp]),
    "hhb_spike_deliver": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp]),
    "hhb_cortex_input_dev": (_i32, [_i32, _i64, _i64, _vp, _i64, _vp, _vp, _dbl, _i32, _vp, _vp, _dbl, _dbl,
                                    C.c_uint64, _i64, _vp, _vp, _dbl, _vp]),
    "hhb_spike_deliver_dev": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp]),
    "hhb_cortex_tick": (_i32, [_vp, _vp]),
    "hhb_spike_event_counts": (_i32, [_i64, _i64, _vp, _i64, _vp, _vp]),
    "hhb_spike_events": (_i32, [_i64, _i64, _vp, _i64, _vp, _vp, _vp, _vp]),
    "hhb_cortex_run": (_i32, [C.POINTER(Params), _i64, _i64, _i64, _i64, _vp, _vp, _dbl, _i32, _vp, _dbl, _dbl,
                              C.c_uint64, _i64, _dbl, _vp, _vp, _i64, _vp, _i32, _i64, _vp, _i64, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp]),
    "hhb_cortex_run_ex": (_i32, [C.POINTER(Params), _i64, _i64, _i64, _i64, _vp, _vp, _dbl, _i32, _vp, _dbl, _dbl,
                                 C.c_uint64, _i64, _dbl, _vp, _vp, _i64, _vp, _i32, _i64, _vp, _i64, _vp, _vp, _vp,
                                 _vp, _vp, _vp, C.POINTER(Thalamic), _vp]),
    "hhb_thalamic_drive": (_i32, [_i32, _i64, _i64, _vp, C.POINTER(Thalamic), _vp, _vp]),
    "hhb_cortex_run_replicas": (_i32, [C.POINTER(Params), _i64, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _dbl, _i32, _vp, _dbl, _dbl,
                              C.c_uint64, _i64, _dbl, _vp, _vp, _i64, _vp, _i32, _i64, _vp, _i64, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp]),
    "hhb_scale_f32": (_i32, [_i64, _vp, _vp, _dbl, _vp, _vp]),
    "hhb_psp_filter": (_i32, [_i32, _i64, _i64, _i32, _vp, _vp, _vp, _vp]),
    "hhb_readout_drive": (_i32, [_i32, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "hhb_readout_workspace": (_i64, [_i32, _i64]),
    "hhb_readout_grad": (_i32, [_i32, _i64, _i64, _i64, _vp, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "hhb_lif_forward": (_i32, [_i32, _i64, _i64, _dbl, _dbl, _dbl, _dbl, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _vp]),
    "hhb_lif_backward": (_i32, [_i32, _i64, _dbl, _dbl, _dbl, _dbl, C.POINTER(Surrogate), _vp, _vp, _i64, _vp, _vp,
                                _vp, _vp, _vp, _vp]),
    "hhb_morph_forward": (_i32, [_i32, _i32, _vp, _i32, _vp, _i32, _vp, _vp, _vp, _i64, _i64,
                                 _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _vp]),
    "hhb_spike_deliver_flat": (_i32, [_i64, _vp, _vp, _vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _vp, _vp]),
    "hhb_spike_scratch": (_i64, [_i64]),
    "hhb_cortex_step_batch": (_i32, [_i32, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _dbl, _vp, _dbl, _dbl, C.c_uint64,
                                     _vp, _dbl, _vp, _vp, _vp, _vp, _vp, _vp, _i32, _vp]),
    "hhb_jit_status": (C.c_char_p, []),
    "hhb_jit_source": (_i64, [C.POINTER(Params), C.c_char_p, _i64]),
    "hhb_jit_cubin": (_i64, [C.POINTER(Params), _i32, _vp, _i64]),
}

_lock = threading.Lock()
_lib = None
_load_error: str | None = None


def load():
    """Load and type the library once; raise NativeLibraryError if unusable."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            _load_error = (f"{LIB_PATH} not built; run `python -m paper_2601_21407_b200._build` "
                           "(there is no CPU fallback)")
            raise NativeLibraryError(_load_error)
        try:
            lib = C.CDLL(LIB_PATH)
        except OSError as e:
            raise NativeLibraryError(f"cannot load {LIB_PATH}: {e}") from None
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.hhb_abi_version() != ABI_VERSION:
            raise NativeLibraryError("libhhb200.so ABI version mismatch; rebuild")
        _lib = lib
        return lib


def check(rc: int, what: str):
    if rc == OK:
        return
    msg = load().hhb_last_error().decode(errors="replace")
    if rc == EINVAL:
        raise UsageError(f"{what}: {msg}")
    raise NativeLibraryError(f"{what} failed (code {rc}): {msg}")


def pack_rate(fn) -> Rate:
    return Rate(RATE_KIND[fn.kind], 0, float(fn.a), float(fn.v0), float(fn.b))


def pack_gate(gate, channel: int = 0) -> Gate:
    return Gate(pack_rate(gate.alpha), pack_rate(gate.beta), int(gate.exponent), channel)


def pack_params(channels, c_m=1.0, dt=1.0, v_theta=0.0, v_rest=-65.0, rate_scale=1.0) -> Params:
    """Flatten a channel list (HHParams.channels) into the C table."""
    P = Params()
    gi = 0
    if len(channels) > MAX_CHANNELS:
        raise ConfigurationError(f"at most {MAX_CHANNELS} channels are supported, got {len(channels)}")
    for ci, ch in enumerate(channels):
        P.channels[ci] = Channel(float(ch.g_max), float(ch.e_rev), gi, len(ch.gates))
        for g in ch.gates:
            if gi >= MAX_GATES:
                raise ConfigurationError(f"at most {MAX_GATES} gates are supported")
            P.gates[gi] = pack_gate(g, ci)
            gi += 1
    P.n_gates = gi
    P.n_channels = len(channels)
    P.c_m, P.dt, P.v_theta, P.v_rest, P.rate_scale = (float(c_m), float(dt), float(v_theta),
                                                        float(v_rest), float(rate_scale))
    lib = load()
    if lib.hhb_check_params(C.byref(P)) != OK:
        raise ConfigurationError(lib.hhb_last_error().decode(errors="replace"))
    return P


def pack_hh(params) -> Params:
    return pack_params(params.channels, params.c_m, params.dt, params.v_theta, params.v_rest,
                       params.rate_scale)


def pack_surrogate(spec) -> Surrogate:
    return Surrogate(SUR_KIND[spec.kind], 0, float(spec.width))


def jit_cubin(params, kind: int = 0) -> bytes:
    """Compile-only NVRTC build of a generated module (0: forward + backward,
    1: persistent network kernel, 2: its 4-replica variant) -> sm_100a cubin
    bytes.  Needs libnvrtc only (no GPU)."""
    lib = load()
    P = pack_hh(params)
    n = int(lib.hhb_jit_cubin(C.byref(P), kind, None, 0))
    if n < 0:
        raise NativeLibraryError(lib.hhb_last_error().decode(errors="replace"))
    buf = C.create_string_buffer(n)
    lib.hhb_jit_cubin(C.byref(P), kind, buf, n)
    return buf.raw[:n]


def jit_source(params) -> str:
    """CUDA source the library generates for `params` (float kernels)."""
    P = pack_hh(params)
    lib = load()
    n = int(lib.hhb_jit_source(C.byref(P), None, 0))
    buf = C.create_string_buffer(n)
    lib.hhb_jit_source(C.byref(P), buf, n)
    return buf.value.decode()


def jit_status() -> str:
    return load().hhb_jit_status().decode()
