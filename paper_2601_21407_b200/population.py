"""Device-resident HH populations advanced in time chunks.

`simulate` (dynamics.py:541-586) materialises the whole (T, n) current and
voltage series.  At BASELINE config 2 (10M neurons x 10,000 steps) that is
400 GB per series in fp32, more than one B200 holds, so this module runs the
same computation chunk by chunk: the neuron state stays on the device across
chunks (bit-identical to a one-shot simulate: the kernel is restartable, see
tests/test_gpu_forward.py::test_chunked_simulation_equals_one_shot), each
chunk's stimulus is produced on the device, and each chunk's trace (V and the
spike bitmap) is written to a reused buffer the caller can consume.

Launches per chunk: one hhb_forward_poisson when the stimulus is the
Poisson drive (drawn in registers inside the forward kernel), otherwise the
stimulus fill plus one hhb_forward.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from .dynamics import HHParams, _forward, _raise_if_bad, _table, init_state


class PoissonCurrent:
    """I[t, j] = amp * Poisson(lam), drawn on the device by Philox-4x32-10 keyed
    by (seed, global neuron id, global step): shards of a population and
    chunks of a run draw exactly the numbers an unsharded one-shot run draws.
    BASELINE config 2 uses amp = 2.0, lam = 2.0."""

    def __init__(self, lam: float = 2.0, amp: float = 2.0, seed: int = 0):
        self.lam, self.amp, self.seed = float(lam), float(amp), int(seed)

    def fill(self, out: torch.Tensor, step_base: int, neuron_base: int = 0) -> int:
        steps, n = out.shape
        nat.check(nat.load().hhb_poisson_current(
            D.code(out.dtype), n, steps, self.seed, neuron_base, step_base, self.lam, self.amp,
            out.data_ptr(), out.stride(0), D.stream()), "poisson current")
        return 1  # kernel launches


class Population:
    """n HH neurons on one device, stepped `chunk` steps per launch.

    neuron_base offsets the global neuron ids (for the stimulus keying) when
    the population is one shard of a larger one.
    """

    def __init__(self, params: HHParams, n: int, chunk: int = 100, device=None,
                 record_v: bool = True, record_spikes: bool = True, neuron_base: int = 0,
                 fuse_stimulus: bool = True):
        self.params = params
        # PoissonCurrent is drawn inside the forward kernel (hhb_forward_poisson)
        # unless fuse_stimulus=False, which writes it to i_buf first
        self.fuse_stimulus = bool(fuse_stimulus)
        self.n = int(n)
        self.chunk = int(chunk)
        self.neuron_base = int(neuron_base)
        dev = device or D.require_cuda()
        self.device = dev
        st = init_state(params, (self.n,), device=dev)
        self.v, self.g = st.v, st.gates
        td = D.torch_dtype(params.dtype)
        self.i_buf = None if self.fuse_stimulus else torch.empty((self.chunk, self.n), dtype=td, device=dev)
        self.v_buf = torch.empty((self.chunk, self.n), dtype=td, device=dev) if record_v else None
        words = (self.n + 31) // 32
        self.bits = torch.empty((self.chunk, words), dtype=torch.int32, device=dev) if record_spikes else None
        self.first_bad = torch.empty(1, dtype=torch.int64, device=dev)
        self.t = 0
        self.launches = 0

    def reset(self):
        st = init_state(self.params, (self.n,), device=self.device)
        self.v.copy_(st.v)
        self.g.copy_(st.gates)
        self.t = 0

    def advance(self, stimulus, steps: int, on_chunk=None, check: bool = False, events=None):
        """Run `steps` steps.  stimulus: PoissonCurrent or a callable
        fill(out, step_base, neuron_base).  on_chunk(t0, v_buf, bits) is called
        after each chunk is enqueued.  events: optional list collecting
        (start, mid, end) CUDA events per chunk (stimulus / forward split)."""
        done = 0
        self.first_bad.fill_(D.INT64_MAX)
        while done < steps:
            tc = min(self.chunk, steps - done)
            e0 = e1 = e2 = None
            if events is not None:
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
            fused = self.fuse_stimulus and isinstance(stimulus, PoissonCurrent)
            if not fused:
                if self.i_buf is None:
                    self.i_buf = torch.empty((self.chunk, self.n), dtype=D.torch_dtype(self.params.dtype),
                                             device=self.device)
                cur = self.i_buf[:tc]
                self.launches += stimulus.fill(cur, self.t, self.neuron_base)
            if events is not None:
                e1.record()
            v_out = None if self.v_buf is None else self.v_buf[:tc]
            bits = None if self.bits is None else self.bits[:tc]
            if fused:
                words = (self.n + 31) // 32
                nat.check(nat.load().hhb_forward_poisson(
                    C.byref(_table(self.params)), D.code(self.params.dtype), self.n, tc,
                    self.v.data_ptr(), D.ptr(self.g) if self.g.numel() else None, self.n,
                    self.v.data_ptr(), D.ptr(self.g) if self.g.numel() else None,
                    stimulus.seed, self.neuron_base, stimulus.lam, stimulus.amp,
                    D.ptr(v_out), self.n, D.ptr(bits), words, None, 1, self.n,
                    self.t, self.first_bad.data_ptr(), D.stream()), "hhb_forward_poisson")
            else:
                _forward(self.params, self.v, self.g, cur, self.n, 1, tc, v_fin=self.v, g_fin=self.g,
                         v_out=v_out, bits=bits, step_base=self.t, first_bad=self.first_bad,
                         reset_bad=False)
            self.launches += 1
            if events is not None:
                e2.record()
                events.append((e0, e1, e2))
            if check:
                _raise_if_bad(self.first_bad)
            if on_chunk is not None:
                on_chunk(self.t, None if self.v_buf is None else self.v_buf[:tc],
                         None if self.bits is None else self.bits[:tc])
            self.t += tc
            done += tc
        return self
