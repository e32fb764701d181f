"""Host-buffer path of `simulate` (numpy in, numpy out) as a copy/compute
pipeline.

The reference's `simulate` (dynamics.py:541-586) takes a host (T,)+S current
series and returns host float64 V and bool spike series.  For a large call the
cost is the PCIe traffic, so the series is cut into time chunks and three
things overlap: worker threads copy (and cast) chunk k+1 of the caller's
array into a pinned staging buffer and a copy stream moves it to the device,
the compute stream runs the fused forward kernel on chunk k (state carried in
registers -> device buffers between launches, bit-identical to one launch),
casts V to float64 and unpacks the spike bitmap, and a second copy stream
moves chunk k-1 into the output arrays, which live in pinned memory so the DMA
writes them directly.
"""

from __future__ import annotations

import concurrent.futures as cf
import os

import numpy as np
import torch

from . import _device as D

_POOL = None


def _pool():
    global _POOL
    if _POOL is None:
        _POOL = cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4))
    return _POOL


def _par_copy(dst: np.ndarray, src: np.ndarray):
    """dst[...] = src (with dtype cast), split over worker threads; NumPy
    releases the GIL inside the copy loop.  Contiguous arrays are split by
    elements (a one-row chunk still uses every thread), others by rows."""
    workers = _pool()._max_workers
    if dst.size < (1 << 20) or workers <= 1:
        np.copyto(dst, src, casting="unsafe")
        return
    if dst.flags.c_contiguous and src.flags.c_contiguous and dst.shape == src.shape:
        d, s_ = dst.reshape(-1), src.reshape(-1)
        step = (d.size + workers - 1) // workers
        step = (step + 1023) & ~1023
        futs = [_pool().submit(np.copyto, d[a:a + step], s_[a:a + step], "unsafe") for a in range(0, d.size, step)]
    else:
        rows = dst.shape[0]
        step = (rows + workers - 1) // workers
        futs = [_pool().submit(np.copyto, dst[a:a + step], src[a:a + step], "unsafe") for a in range(0, rows, step)]
    for f in futs:
        f.result()


def pinned_empty(shape, dtype) -> np.ndarray:
    """A numpy array backed by page-locked memory (kept alive by the array)."""
    t = torch.empty(shape, dtype={np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32,
                                  np.dtype(bool): torch.bool}[np.dtype(dtype)], pin_memory=True)
    return t.numpy()


CHUNK_BYTES = int(os.environ.get("HHB_PIPE_CHUNK_MB", "64")) << 20   # input bytes per pipelined chunk
MIN_CHUNKS = int(os.environ.get("HHB_PIPE_MIN_CHUNKS", "12"))         # chunks of a long, narrow call (measured: 12-16 best for config 1)


def simulate_host(params, i2: np.ndarray, v: torch.Tensor, g: torch.Tensor, forward, unpack,
                  chunk_bytes: int | None = None):
    """Run the forward over host array i2 (T, n) in pipelined chunks.

    forward(cur, tc, v_out, bits, step_base) enqueues one launch on the current
    stream; unpack(bits, tc, n, out_u8) likewise.  Returns (V float64 (T, n),
    spikes bool (T, n)) as pinned-backed numpy arrays.
    """
    T, n = i2.shape
    dev = v.device
    chunk_bytes = CHUNK_BYTES if chunk_bytes is None else chunk_bytes
    cdt = D.np_dtype(params.dtype)
    tdt = D.torch_dtype(cdt)
    tc_max = int(max(1, min(T, chunk_bytes // max(1, n * cdt.itemsize))))
    # small populations over long horizons (config 1: 1,024 x 10,000) fit one
    # chunk: cut them into >= MIN_CHUNKS so the copies overlap the
    # (latency-bound) compute
    if T >= 4 * 64 and tc_max * MIN_CHUNKS > T:
        tc_max = max(64, (T + MIN_CHUNKS - 1) // MIN_CHUNKS)
    nbuf = 2
    stage = [torch.empty((tc_max, n), dtype=tdt, pin_memory=True) for _ in range(nbuf)] \
        if not (i2.dtype == cdt and i2.flags.c_contiguous and torch.from_numpy(i2).is_pinned()) else None
    d_in = [torch.empty((tc_max, n), dtype=tdt, device=dev) for _ in range(nbuf)]
    d_v = [torch.empty((tc_max, n), dtype=tdt, device=dev) for _ in range(nbuf)]
    d_v64 = [torch.empty((tc_max, n), dtype=torch.float64, device=dev) for _ in range(nbuf)]
    d_bits = [torch.empty((tc_max, (n + 31) // 32), dtype=torch.int32, device=dev) for _ in range(nbuf)]
    d_spk = [torch.empty((tc_max, n), dtype=torch.uint8, device=dev) for _ in range(nbuf)]
    out_v = pinned_empty((T, n), np.float64)
    out_s = pinned_empty((T, n), bool)
    tv = torch.from_numpy(out_v)
    ts = torch.from_numpy(out_s.view(np.uint8))

    compute = torch.cuda.current_stream(dev)
    h2d = torch.cuda.Stream(dev)
    d2h = torch.cuda.Stream(dev)
    ev_staged = [None] * nbuf      # H2D finished reading stage[b]
    ev_loaded = [None] * nbuf      # d_in[b] holds its chunk
    ev_computed = [None] * nbuf    # d_v64/d_spk[b] hold results
    ev_drained = [None] * nbuf     # D2H finished reading d_v64/d_spk[b]

    chunks = [(t0, min(T, t0 + tc_max)) for t0 in range(0, T, tc_max)]

    # a caller's array already in page-locked memory (and of the compute dtype)
    # is DMA'd as it is: no staging copy through host memory
    src_t = torch.from_numpy(i2) if (i2.dtype == cdt and i2.flags.c_contiguous) else None
    direct = src_t is not None and src_t.is_pinned()

    def stage_and_load(k):
        t0, t1 = chunks[k]
        b = k % nbuf
        if not direct:
            if ev_staged[b] is not None:
                ev_staged[b].synchronize()      # stage[b] free again
            _par_copy(stage[b][:t1 - t0].numpy(), i2[t0:t1])
        with torch.cuda.stream(h2d):
            if ev_computed[b] is not None:
                h2d.wait_event(ev_computed[b])  # d_in[b] consumed by the forward
            d_in[b][:t1 - t0].copy_(src_t[t0:t1] if direct else stage[b][:t1 - t0], non_blocking=True)
            ev_staged[b] = torch.cuda.Event()
            ev_staged[b].record(h2d)
            ev_loaded[b] = ev_staged[b]

    stage_and_load(0)
    for k, (t0, t1) in enumerate(chunks):
        b = k % nbuf
        tc = t1 - t0
        compute.wait_event(ev_loaded[b])
        if ev_drained[b] is not None:
            compute.wait_event(ev_drained[b])   # outputs of chunk k-2 copied out
        forward(d_in[b][:tc], tc, d_v[b][:tc], d_bits[b][:tc], t0)
        d_v64[b][:tc].copy_(d_v[b][:tc])
        unpack(d_bits[b][:tc], tc, n, d_spk[b][:tc])
        ev_computed[b] = torch.cuda.Event()
        ev_computed[b].record(compute)
        with torch.cuda.stream(d2h):
            d2h.wait_event(ev_computed[b])
            tv[t0:t1].copy_(d_v64[b][:tc], non_blocking=True)
            ts[t0:t1].copy_(d_spk[b][:tc], non_blocking=True)
            ev_drained[b] = torch.cuda.Event()
            ev_drained[b].record(d2h)
        if k + 1 < len(chunks):
            stage_and_load(k + 1)               # host copy overlaps the kernel
    d2h.synchronize()
    compute.synchronize()
    if TRACE:
        print(f"[pipeline] T={T} n={n} chunks={len(chunks)} x {tc_max} steps", flush=True)
    return out_v, out_s


TRACE = bool(int(os.environ.get("HHB_PIPE_TRACE", "0")))
