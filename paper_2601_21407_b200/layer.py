"""Differentiable HH SNN layer: dense synaptic projection on tcgen05 + HH
population + surrogate-gradient BPTT.

This is the composition of the reference's readout pipeline
(`ReadoutModel.forward/grads`, learn.py:238-274: DenseLayer -> simulate ->
backward_through_time -> einsum) generalised from one output neuron to
`n_out`, as BASELINE configs 3 and 4 use it:

  forward   I[t, b, :] = bf16(x[t, b, :]) . bf16(W)^T + bias     (hhb_gemm, bf16)
            V, spikes  = HH(I) over T steps, checkpoints every K    (hhb_forward)
  backward  dI        = BPTT(dL/dV, dL/dspikes)                      (hhb_backward)
            dW        = dI^T . bf16(x)     dX = dI . bf16(W)         (hhb_gemm, bf16x2)
            db        = column sums of dI                            (hhb_col_sum)

The gradient GEMMs split the fp32 dI into bf16 hi + lo and fold both products
into one GEMM with K doubled, so the bf16 tensor cores carry ~16 mantissa bits
of dI (plain tf32 operands measured 8e-4 normwise error against the 1e-3
contract; tools/gemm_err.py).  Saved for backward: bf16 x and W, the fp32
current and the HH checkpoints -- not the V history.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np
import torch

from . import _device as D
from . import _native as nat
from .adjoint import SurrogateSpec, _backward, default_surrogate, make_plan
from .defaults import cortical_rs_params
from .dynamics import HHParams, _forward, _raise_if_bad, _table, _unpack, steady_state_gates
from .errors import GradientOverflowError, UsageError

BF16, TF32 = 0, 1

# Per-component kernel timing for bench.py's roofline (off by default):
# when TIMERS is a dict, each component records CUDA events on the stream it
# runs on -- TIMERS[name] = [(start, end, units), ...] with units the
# neuron-steps (HH kernels) or FLOPs (GEMMs) of that launch.
TIMERS = None


class _timed:
    def __init__(self, name: str, units: float):
        self.name, self.units = name, units

    def __enter__(self):
        if TIMERS is not None:
            # keep the GPU busy (~0.5 ms spin) while the host prepares the
            # component's launch, so the start event brackets the kernel only
            torch.cuda._sleep(1_000_000)
            self.e0 = torch.cuda.Event(enable_timing=True)
            self.e0.record()
        return self

    def __exit__(self, *exc):
        if TIMERS is not None:
            e1 = torch.cuda.Event(enable_timing=True)
            e1.record()
            TIMERS.setdefault(self.name, []).append((self.e0, e1, self.units))
        return False


def _pad8(k: int) -> int:
    return (k + 7) // 8 * 8


def _stream():
    return torch.cuda.current_stream().cuda_stream


def gemm(A: torch.Tensor, B: torch.Tensor, K: int, bias=None, out=None, splits: int | None = None):
    """out[M][N] = A[:, :K] . B[:, :K]^T (+ bias) with bf16 operands (row pitch = stride(0))."""
    M, N = A.shape[0], B.shape[0]
    if out is None:
        out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    lib = nat.load()
    if splits is None:
        splits = 0          # the library picks the split count for its tile grid
    ws_n = int(lib.hhb_gemm_workspace(M, N, splits if splits > 0 else 32))
    ws = _workspace(ws_n, A.device) if ws_n else None
    nat.check(lib.hhb_gemm(BF16, M, N, K, A.data_ptr(), A.stride(0), B.data_ptr(), B.stride(0),
                           D.ptr(bias), out.data_ptr(), out.stride(0), splits, D.ptr(ws), _stream()), "hhb_gemm")
    return out


def to_bf16_padded(x2: torch.Tensor) -> torch.Tensor:
    """(rows, k) fp32 -> (rows, pad8(k)) bf16, zero tail (TMA needs 16 B pitches)."""
    rows, k = x2.shape
    kp = _pad8(k)
    if kp == k and x2.is_contiguous():
        out = torch.empty((rows, k), dtype=torch.bfloat16, device=x2.device)
        nat.check(nat.load().hhb_cast_bf16(x2.numel(), x2.data_ptr(), out.data_ptr(), _stream()), "cast")
        return out
    out = torch.zeros((rows, kp), dtype=torch.bfloat16, device=x2.device)
    out[:, :k] = x2.to(torch.bfloat16)
    return out


def split3_padded(x2: torch.Tensor, order: int) -> tuple[torch.Tensor, int]:
    """(rows, k) fp32 -> (rows, 3 kp) bf16 slots (kp = pad8(k)): order 0
    [hi | lo | hi], order 1 [hi | hi | lo] (hhb_split3_bf16).  Returns the
    buffer and the slot width kp."""
    rows, k = x2.shape
    kp = _pad8(k)
    alloc = torch.empty if kp == k else torch.zeros
    out = alloc((rows, 3 * kp), dtype=torch.bfloat16, device=x2.device)
    nat.check(nat.load().hhb_split3_bf16(rows, k, x2.data_ptr(), x2.stride(0), out.data_ptr(), 3 * kp, kp, order,
                                         _stream()), "split3")
    return out, kp


def grad_weight(dI: torch.Tensor, xb: torch.Tensor, k_in: int) -> torch.Tensor:
    """dW[N][k_in] = dI^T . xb  (dI (M, N) fp32, xb (M, >=k_in) bf16), bf16x2."""
    M, N = dI.shape
    lib = nat.load()
    m2 = 2 * M
    ld = _pad8(m2)
    a = torch.empty((N, ld), dtype=torch.bfloat16, device=dI.device)
    b = torch.empty((k_in, ld), dtype=torch.bfloat16, device=dI.device)
    nat.check(lib.hhb_transpose(3, M, N, dI.data_ptr(), dI.stride(0), a.data_ptr(), ld, _stream()), "split^T")
    nat.check(lib.hhb_transpose(4, M, k_in, xb.data_ptr(), xb.stride(0), b.data_ptr(), ld, _stream()), "dup^T")
    return gemm(a, b, m2)


def grad_input(dI: torch.Tensor, wb: torch.Tensor, k_in: int) -> torch.Tensor:
    """dX[M][k_in] = dI . wb  (wb (N, >=k_in) bf16), bf16x2."""
    M, N = dI.shape
    lib = nat.load()
    n2 = 2 * N
    ld = _pad8(n2)
    a = torch.empty((M, ld), dtype=torch.bfloat16, device=dI.device)
    b = torch.empty((k_in, ld), dtype=torch.bfloat16, device=dI.device)
    nat.check(lib.hhb_split_rows_bf16(M, N, dI.data_ptr(), dI.stride(0), a.data_ptr(), ld, _stream()), "split")
    nat.check(lib.hhb_transpose(4, N, k_in, wb.data_ptr(), wb.stride(0), b.data_ptr(), ld, _stream()), "dup^T")
    return gemm(a, b, n2)


def gemm_ex(flags: int, M: int, N: int, K: int, A: torch.Tensor, A2, lda: int, B: torch.Tensor, ldb: int,
            splits: int | None = None) -> torch.Tensor:
    """out[M][N] = (A + A2) . B^T with MN-major operands where flags say so (hhb_gemm_ex)."""
    out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    lib = nat.load()
    if splits is None:
        splits = 0          # the library picks the split count for its tile grid
    ws_n = int(lib.hhb_gemm_workspace(M, N, splits if splits > 0 else 32))
    ws = _workspace(ws_n, A.device) if ws_n else None
    nat.check(lib.hhb_gemm_ex(flags, M, N, K, A.data_ptr(), D.ptr(A2), lda, B.data_ptr(), ldb, None,
                              out.data_ptr(), N, splits, D.ptr(ws), _stream()), "hhb_gemm_ex")
    return out


def gemm_ex2(flags: int, M: int, N: int, K: int, A: torch.Tensor, A2: torch.Tensor, lda: int, B: torch.Tensor,
             ldb: int, k_switch: int, splits: int | None = None) -> torch.Tensor:
    """out[M][N] = [A | A2] . B^T: K-major A for k < k_switch, A2 (same lda) at
    k - k_switch above (hhb_gemm_ex2)."""
    out = torch.empty((M, N), dtype=torch.float32, device=A.device)
    lib = nat.load()
    if splits is None:
        splits = 0
    ws_n = int(lib.hhb_gemm_workspace(M, N, splits if splits > 0 else 32))
    ws = _workspace(ws_n, A.device) if ws_n else None
    nat.check(lib.hhb_gemm_ex2(flags, M, N, K, A.data_ptr(), A2.data_ptr(), lda, B.data_ptr(), ldb, None,
                               out.data_ptr(), N, splits, D.ptr(ws), k_switch, _stream()), "hhb_gemm_ex2")
    return out


_WS = {}


def _workspace(n: int, dev) -> torch.Tensor:
    """Split-K scratch, kept per device and stream (grows; the stream orders
    its reuse; the side stream of overlapped weight gradients has its own)."""
    key = (str(dev), torch.cuda.current_stream(dev).cuda_stream)
    w = _WS.get(key)
    if w is None or w.numel() < n:
        w = torch.empty(n, dtype=torch.float32, device=dev)
        _WS[key] = w
    return w


A_MN, B_MN = 1, 2


def col_sum_f32(src: torch.Tensor) -> torch.Tensor:
    """Column sums of a (rows, cols) fp32 matrix as fp32, fixed order, one
    launch for rows <= 512 (hhb_col_sum_ex)."""
    M, N = src.shape
    lib = nat.load()
    out = torch.empty(N, dtype=torch.float32, device=src.device)
    scratch = (torch.empty(max(1, int(lib.hhb_col_sum_scratch(M, N))), dtype=torch.float64, device=src.device)
               if M > 512 else None)
    nat.check(lib.hhb_col_sum_ex(M, N, src.data_ptr(), src.stride(0), None, out.data_ptr(), D.ptr(scratch),
                                 _stream()), "colsum")
    return out


def col_sum(dI: torch.Tensor) -> torch.Tensor:
    M, N = dI.shape
    lib = nat.load()
    out = torch.zeros(N, dtype=torch.float64, device=dI.device)
    scratch = torch.empty(max(1, int(lib.hhb_col_sum_scratch(M, N))), dtype=torch.float64, device=dI.device)
    nat.check(lib.hhb_col_sum(M, N, dI.data_ptr(), dI.stride(0), out.data_ptr(), scratch.data_ptr(), _stream()),
              "colsum")
    return out


def _layer_grads(layer, xb, wb, cur, ckpt, K, shape, x_requires_grad, sv, ss, sv_ld=None, sv_scale=None):
    """BPTT of the layer's HH population from seeds (sv, ss) and the projection
    gradients (dX, dW, db)."""
    T, B, k_in, n_out = shape
    M, n = T * B, B * n_out
    p = layer.params
    # adjoint state (d_v, d_gates) and the per-neuron dI sums: one zeroed block
    zb = torch.zeros((2 + p.n_gates) * n, dtype=torch.float32, device=cur.device)
    adj_v = zb[:n]
    adj_g = zb[n:(1 + p.n_gates) * n].view(p.n_gates, n)
    # dI leaves the BPTT kernel as bf16 hi/lo halves in one buffer, row (t, b) =
    # [hi (P) | lo (P)] (P = n_out padded to 8 for TMA pitches), + per-neuron
    # sums; the gradient GEMMs read it (and X, W) in place: MN-major hi / lo
    # planes at lda = 2P for dW, K-major [hi | lo] rows for dX
    P = _pad8(n_out)
    # (pad columns n_out..P of each half are read by the K-concatenated dX GEMMs: zeros)
    H = (torch.empty if P == n_out else torch.zeros)((T, B * 2 * P), dtype=torch.bfloat16, device=cur.device)
    hi, lo = H, H.view(-1)[P:]
    dsum = zb[(1 + p.n_gates) * n:]
    with _timed("hh_bptt", T * n):
        _, d_params, gbad = _backward(p, layer.surrogate, cur, n, 1, T, n, ckpt, K, sv, ss, adj_v, adj_g,
                                      want_d_i=False, split=(hi, lo, n_out, 2 * P), d_sum=dsum, ck_ld=n,
                                      sv_ld=sv_ld, sv_scale=sv_scale)
    layer._last_gbad = gbad
    if layer.check_finite:
        b = int(gbad.item())
        if b >= 0:
            raise GradientOverflowError("adjoint state became non-finite", b)
    layer.param_grads = d_params                       # {d_c_m, d_g_max[...]} (fp64, device)
    x3 = layer.proj == "bf16x3"
    kp = _pad8(k_in) if x3 else 0           # slot width of the [x_hi | x_lo (| x_hi)] rows

    def weight_grad():
        # dW[j][k] = sum_m dI[m][j] X[m][k]: A = dI^T, B = X^T, both MN-major views;
        # bf16x3: (dI_hi + dI_lo) . x_hi + dI_hi . x_lo (slots 0 and 1 of xb)
        with _timed("grad_w", 2.0 * M * n_out * k_in):
            if xb.dtype == torch.float32:
                # the fp32 x itself (_fused_dw): rounded (bf16x3: and split) on chip, one GEMM
                lib = nat.load()
                dW = torch.empty((n_out, k_in), dtype=torch.float32, device=xb.device)
                ws_n = int(lib.hhb_gemm_workspace(n_out, k_in, 32))
                ws = _workspace(ws_n, xb.device) if ws_n else None
                nat.check(lib.hhb_gemm_f32b(n_out, k_in, M, hi.data_ptr(), lo.data_ptr(), 2 * P, xb.data_ptr(),
                                            xb.stride(0), 1 if x3 else 0, dW.data_ptr(), k_in, 0, D.ptr(ws),
                                            _stream()),
                          "hhb_gemm_f32b")
                return dW
            dW = gemm_ex(A_MN | B_MN, n_out, k_in, M, hi, lo, 2 * P, xb, xb.stride(0))
            if x3:
                dW += gemm_ex(A_MN | B_MN, n_out, k_in, M, hi, None, 2 * P, xb[:, kp:], xb.stride(0))
        return dW

    if layer.overlap_weight_grad:
        # dW, db on a side stream: they overlap the previous layer's BPTT (CUDA
        # cores vs tensor cores); the grads are handed over when the backward
        # pass ends (autograd engine callback: the main stream waits, then
        # .grad is set or accumulated), so autograd gets None for them here
        main = torch.cuda.current_stream(cur.device)
        side = _side_stream(cur.device)
        fork = torch.cuda.Event()
        fork.record(main)
        side.wait_event(fork)
        with torch.cuda.stream(side):
            dW = weight_grad()
            db = col_sum_f32(dsum.view(B, n_out))
            done = torch.cuda.Event()
            done.record(side)
        for t in (hi, lo, zb, xb):
            t.record_stream(side)
        weight, bias = layer.weight, layer.bias

        def hand_over(gw=dW, gb=db):
            cur_stream = torch.cuda.current_stream(gw.device)
            cur_stream.wait_event(done)
            gw.record_stream(cur_stream)
            gb.record_stream(cur_stream)
            for prm, g in ((weight, gw), (bias, gb)):
                if prm.grad is None:
                    prm.grad = g
                else:
                    prm.grad.add_(g)

        torch.autograd.Variable._execution_engine.queue_callback(hand_over)
        dW = db = None
    else:
        dW = weight_grad()
        db = col_sum_f32(dsum.view(B, n_out))
    dX = None
    if x_requires_grad:
        # dX[m][k] = sum_j dI[m][j] W[j][k]: A = dI (K-major), B = W^T (MN-major view of W);
        # bf16x3: (dI_hi + dI_lo) . W_hi + dI_hi . W_lo (slots 0 and 2 of wb)
        with _timed("grad_x", 2.0 * M * n_out * k_in):
            if x3 and (2 * P) % 64 == 0:
                # one GEMM over K = 3P: [dI_hi | dI_lo] (the buffer's rows), then
                # dI_hi again (k_switch), against the stacked [W_hi; W_hi; W_lo]
                dX = gemm_ex2(B_MN, M, k_in, 3 * P, hi, hi, 2 * P, wb, wb.stride(0), 2 * P)
            elif x3:
                dX = gemm_ex(B_MN, M, k_in, 2 * P, hi, None, 2 * P, wb, wb.stride(0))
                dX += gemm_ex(B_MN, M, k_in, n_out, hi, None, 2 * P, wb[2 * P:], wb.stride(0))
            else:
                dX = gemm_ex(B_MN, M, k_in, n_out, hi, lo, 2 * P, wb, wb.stride(0))
        dX = dX.view(T, B, k_in)
    return dX, dW, db


_SIDE: dict = {}


def _side_stream(dev) -> torch.cuda.Stream:
    key = str(dev)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(dev)
    return _SIDE[key]


def _twin(x):
    """The bf16 copy of x an HHLayer(outputs="spikes") below wrote beside its
    fp32 spikes (exactly x in bf16), if it is still current."""
    T, B, k_in = x.shape
    twin = getattr(x, "_hhb_bf16", None)
    if (twin is not None and twin[1] == x._version and tuple(twin[0].shape) == tuple(x.shape)
            and k_in % 8 == 0):
        return twin[0].view(T * B, k_in)
    return None


def _fused_convert(x, layer) -> bool:
    """bf16x3 projection with the fp32 x converted and split on chip inside the
    GEMM (hhb_gemm_f32a): CTA-pair tiles (>= 512 rows), 8-aligned k_in, n_out a
    multiple of 4 (16-byte output rows).  The bf16 projection keeps the separate
    cast: with one (forward) or two (weight gradient) products per k-step the
    conversion is not hidden -- config 3 0.461 -> 0.483 ms, config 4 2.435 ->
    2.48 ms with both GEMMs converting on chip, 0.475 / 2.463 ms with the
    projection writing the converted x back."""
    import os
    T, B, k_in = x.shape
    n_out = layer.weight.shape[0]
    return (layer.proj == "bf16x3" and T * B >= 512 and k_in % 8 == 0 and n_out % 4 == 0
            and os.environ.get("HHB_LAYER_FUSED_SPLIT", "1") != "0")


def _dw_shape_ok(x, layer) -> bool:
    import os
    return (layer.weight.shape[0] >= 512 and x.shape[2] > 128
            and os.environ.get("HHB_LAYER_FUSED_DW", "1") != "0")


def _fused_dw(x, layer) -> bool:
    """With the on-chip conversion in the projection, the weight gradient also
    reads the fp32 x and converts it on chip (hhb_gemm_f32b), so the projection
    need not write the converted x: 256-wide CTA-pair tiles (n_out >= 512,
    k_in > 128)."""
    return _fused_convert(x, layer) and _dw_shape_ok(x, layer)


def _operands(x, weight, layer):
    """bf16 GEMM operands of the projection: (xb, wb_proj, wb_grad, K) --
    wb_grad is the input gradient's B operand (the stacked [W_hi; W_hi; W_lo]
    for bf16x3, W itself for bf16).  Fused (_fused_convert): xb is the
    empty [x_hi | x_lo] buffer the projection GEMM fills while it converts x."""
    T, B, k_in = x.shape
    if layer.proj == "bf16x3":
        # fp32-class projection: I = x_h.W_h + x_l.W_h + x_h.W_l in one bf16 GEMM over 3 kp
        n_out = weight.shape[0]
        with _timed("operand_prep", T * B * k_in):
            if _fused_convert(x, layer):
                kp = _pad8(k_in)
                # the [x_hi | x_lo] the projection GEMM writes for the weight
                # gradient -- none when that GEMM splits the fp32 x itself
                xb = None if _fused_dw(x, layer) else torch.empty((T * B, 2 * kp), dtype=torch.bfloat16,
                                                                    device=x.device)
            else:
                xb, kp = split3_padded(x.reshape(T * B, k_in).float().contiguous(), 0)
            wb, _ = split3_padded(weight.float().contiguous(), 1)
            if not x.requires_grad:
                return xb, wb, wb, 3 * kp        # no input gradient: its stacked operand is not built
            # the input gradient's B operand: rows [W_hi; W_hi; W_lo], each block
            # n_out rows padded to P (MN-major over the reduction index j)
            P = _pad8(n_out)
            w3 = (torch.empty if (P == n_out and kp == k_in) else torch.zeros)(
                (3 * P, kp), dtype=torch.bfloat16, device=x.device)
            wf = weight.float().contiguous()
            nat.check(nat.load().hhb_split3_bf16(n_out, k_in, wf.data_ptr(), k_in, w3.data_ptr(), kp, P, 2,
                                                 _stream()), "split3 stacked")
        return xb, wb, w3, 3 * kp
    xb = _twin(x)
    if xb is not None:
        pass      # spikes of an HHLayer(outputs="spikes") below: exactly x in bf16, no cast pass
    else:
        with _timed("operand_prep", T * B * k_in):
            xb = to_bf16_padded(x.reshape(T * B, k_in).float().contiguous())
    with _timed("operand_prep", weight.numel()):
        wb = to_bf16_padded(weight.float().contiguous())
    return xb, wb, wb, k_in


def _time_chunks(T: int, K: int, work: int):
    """Time chunks of the pipelined projection + forward: HHB_LAYER_CHUNKS
    (default 1: measured slower) pieces, each a multiple of the checkpoint segment K; one chunk
    for small problems (the GEMM tiles would not fill the GPU)."""
    import os
    C = int(os.environ.get("HHB_LAYER_CHUNKS", "1"))
    if C <= 1 or T < 2 * C or work < (1 << 24):
        return [(0, T)]
    tc = -(-T // C)
    tc = -(-tc // K) * K
    return [(t0, min(T, t0 + tc)) for t0 in range(0, T, tc)]


_PROJ: dict = {}


def _proj_stream(dev) -> torch.cuda.Stream:
    key = str(dev)
    if key not in _PROJ:
        _PROJ[key] = torch.cuda.Stream(dev)
    return _PROJ[key]


def _project_forward(x, weight, bias, layer, K, run_forward):
    """Projection GEMM I = x W^T + b followed by the HH forward, pipelined over
    time chunks: the GEMM of chunk c + 1 (a side stream) runs while the
    forward of chunk c (the current stream) consumes the rows of chunk c --
    the forward is sequential in time, so it can start as soon as its first
    steps' currents exist.  run_forward(cur, t0, t1) launches the forward of
    steps [t0, t1).  Returns (xb, wb_grad, cur)."""
    T, B, k_in = x.shape
    n_out = weight.shape[0]
    xb, wb, wg, kk = _operands(x, weight, layer)
    b32 = bias.float().contiguous()
    cur = torch.empty((T * B, n_out), dtype=torch.float32, device=x.device)
    chunks = _time_chunks(T, K, T * B * n_out)
    x32 = x.reshape(T * B, k_in).float().contiguous() if _fused_convert(x, layer) else None
    x3 = layer.proj == "bf16x3"

    def project(r0, r1):
        if x32 is None:
            gemm(xb[r0:r1], wb, kk, bias=b32, out=cur[r0:r1])
            return
        # fp32 x rounded and split on chip; the GEMM also writes x_hi / x_lo
        # into xb for the weight gradient (B = W_hi, B_lo = W_lo: slots 0 / 2 of wb)
        lib = nat.load()
        M = r1 - r0
        kp = _pad8(k_in) if x3 else 0
        ws_n = int(lib.hhb_gemm_workspace(M, n_out, 32))
        ws = _workspace(ws_n, x.device) if ws_n else None
        nat.check(lib.hhb_gemm_f32a(M, n_out, k_in, x32[r0:].data_ptr(), k_in, wb.data_ptr(),
                                    wb[:, 2 * kp:].data_ptr() if x3 else None, wb.stride(0), b32.data_ptr(),
                                    cur[r0:].data_ptr(), n_out, 0, D.ptr(ws),
                                    None if xb is None else xb[r0:].data_ptr(), 0 if xb is None else xb.stride(0),
                                    kp, _stream()),
                  "hhb_gemm_f32a")

    if len(chunks) == 1:
        with _timed("proj_gemm", 2.0 * T * B * k_in * n_out):
            project(0, T * B)
        run_forward(cur, 0, T)
        return (x32 if xb is None else xb), wg, cur
    main = torch.cuda.current_stream(x.device)
    side = _proj_stream(x.device)
    fork = torch.cuda.Event()
    fork.record(main)
    side.wait_event(fork)
    evs = []
    with torch.cuda.stream(side):
        for t0, t1 in chunks:
            with _timed("proj_gemm", 2.0 * (t1 - t0) * B * k_in * n_out):
                project(t0 * B, t1 * B)
            ev = torch.cuda.Event()
            ev.record(side)
            evs.append(ev)
    for t in (wb, b32, cur) + (() if xb is None else (xb,)) + (() if x32 is None else (x32,)):
        t.record_stream(side)
    for (t0, t1), ev in zip(chunks, evs):
        main.wait_event(ev)
        run_forward(cur, t0, t1)
    return (x32 if xb is None else xb), wg, cur


class _HHLayerFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, weight, bias, layer):
        T, B, k_in = x.shape
        n_out = weight.shape[0]
        n = B * n_out
        p = layer.params
        v0, g0 = layer.rest_state(n, x.device)
        K = layer.segment(T)
        nck = (T + K - 1) // K
        ckpt = torch.empty((nck, 1 + p.n_gates, n), dtype=torch.float32, device=x.device)
        want_v, want_s = layer.outputs in ("both", "v"), layer.outputs in ("both", "spikes")
        v_out = torch.empty((T, n), dtype=torch.float32, device=x.device) if want_v else None
        spikes = torch.empty((T, n), dtype=torch.float32, device=x.device) if want_s else None
        # a spikes-only layer feeds a layer above: its bf16 GEMM operand comes
        # straight out of the forward kernel (attached to the spike tensor)
        sb = (torch.empty((T, n), dtype=torch.bfloat16, device=x.device)
              if layer.outputs == "spikes" and n_out % 8 == 0 else None)
        bad = torch.empty(1, dtype=torch.int64, device=x.device)
        state = {}

        def run_forward(cur, t0, t1):
            full = t0 == 0 and t1 == T
            if full:
                vi, gi, vf, gf = v0, g0, None, None
            else:
                if t0 == 0:
                    state["v"], state["g"] = v0.clone(), g0.clone()
                vi = vf = state["v"]
                gi = gf = state["g"]
            with _timed("hh_forward", (t1 - t0) * n):
                _forward(p, vi, gi, cur[t0 * B:t1 * B].view(t1 - t0, n), n, 1, t1 - t0, v_fin=vf, g_fin=gf,
                         v_out=None if v_out is None else v_out[t0:t1],
                         spk_val=None if spikes is None else spikes[t0:t1],
                         ckpt=ckpt[t0 // K:(t1 + K - 1) // K], ckpt_every=K,
                         spk_bf16=None if sb is None else sb[t0:t1], step_base=t0, first_bad=bad,
                         reset_bad=t0 == 0)

        xb, wb, cur = _project_forward(x, weight, bias, layer, K, run_forward)
        layer._last_bad = bad
        if layer.check_finite:
            _raise_if_bad(bad)
        ctx.set_materialize_grads(False)    # an unused output (V or spikes) seeds nothing
        ctx.save_for_backward(xb, wb, cur, ckpt)
        ctx.layer, ctx.K, ctx.shape = layer, K, (T, B, k_in, n_out)
        ctx.x_requires_grad = x.requires_grad
        s_out = spikes.view(T, B, n_out) if want_s else None
        if sb is not None:
            s_out._hhb_bf16 = (sb.view(T, B, n_out), s_out._version)
        return (v_out.view(T, B, n_out) if want_v else None), s_out

    @staticmethod
    def backward(ctx, d_v, d_s):
        xb, wb, cur, ckpt = ctx.saved_tensors
        T, B, k_in, n_out = ctx.shape
        n = B * n_out
        sv = None if d_v is None else d_v.reshape(T, n).float().contiguous()
        ss = None if d_s is None else d_s.reshape(T, n).float().contiguous()
        dX, dW, db = _layer_grads(ctx.layer, xb, wb, cur, ckpt, ctx.K, ctx.shape, ctx.x_requires_grad, sv, ss)
        return dX, dW, db, None


class _HHLayerMSEFn(torch.autograd.Function):
    """MSE(V, 0) of the layer's membrane trace, fused into its kernels: the
    forward kernel accumulates sum V'^2 (per-block fp64 partials, summed in a
    fixed order) and writes no V trace; the backward kernel reads its seed
    2 V' g / numel (learn.py:86-88) straight from the checkpoints -- with full
    storage the state before step t + 1 is V'(t), and the final state goes to
    one extra slot -- scaled on the fly.  Same arithmetic as
    mse(layer(x)[0]).backward() without the V and seed passes."""

    @staticmethod
    def forward(ctx, x, weight, bias, layer):
        T, B, k_in = x.shape
        n_out = weight.shape[0]
        n = B * n_out
        p = layer.params
        ng = p.n_gates
        v0, g0 = layer.rest_state(n, x.device)
        K = layer.segment(T)
        chunks = _time_chunks(T, K, T * B * n_out)
        npart = int(nat.load().hhb_forward_partials(n))
        # one row of fp64 partials per time chunk (each launch writes its own)
        sq = torch.zeros((len(chunks), npart), dtype=torch.float64, device=x.device)
        if K == 1:
            ckpt = torch.empty((T + 1, 1 + ng, n), dtype=torch.float32, device=x.device)
            v_out = None
        else:
            ckpt = torch.empty(((T + K - 1) // K, 1 + ng, n), dtype=torch.float32, device=x.device)
            v_out = torch.empty((T, n), dtype=torch.float32, device=x.device)
        bad = torch.empty(1, dtype=torch.int64, device=x.device)
        state = {}

        def run_forward(cur, t0, t1):
            c = [i for i, ch in enumerate(chunks) if ch[0] == t0][0] if len(chunks) > 1 else 0
            if t0 == 0:
                state["v"], state["g"] = (v0, g0) if t1 == T else (v0.clone(), g0.clone())
            vi, gi = state["v"], state["g"]
            if K == 1 and t1 == T:
                vf, gf = ckpt[T, 0], ckpt[T, 1:]        # the final state goes to the extra slot
            else:
                vf, gf = vi, gi
            with _timed("hh_forward", (t1 - t0) * n):
                _forward(p, vi, gi, cur[t0 * B:t1 * B].view(t1 - t0, n), n, 1, t1 - t0, v_fin=vf, g_fin=gf,
                         v_out=None if v_out is None else v_out[t0:t1],
                         ckpt=ckpt[t0 // K:(t1 + K - 1) // K], ckpt_every=K, sq_part=sq[c], step_base=t0,
                         first_bad=bad, reset_bad=t0 == 0)

        xb, wb, cur = _project_forward(x, weight, bias, layer, K, run_forward)
        layer._last_bad = bad
        if layer.check_finite:
            _raise_if_bad(bad)
        ctx.save_for_backward(xb, wb, cur, ckpt, v_out)
        ctx.layer, ctx.K, ctx.shape = layer, K, (T, B, k_in, n_out)
        ctx.x_requires_grad = x.requires_grad
        loss = torch.empty((), dtype=torch.float32, device=x.device)
        nat.check(nat.load().hhb_sum_f64(sq.numel(), sq.data_ptr(), 1.0 / (T * n), None, loss.data_ptr(), _stream()),
                  "loss")
        return loss

    @staticmethod
    def backward(ctx, g):
        xb, wb, cur, ckpt, v_out = ctx.saved_tensors
        T, B, k_in, n_out = ctx.shape
        n = B * n_out
        scale = (g.float() * (2.0 / (T * n))).reshape(1).contiguous()
        if ctx.K == 1:
            seed, sv_ld = ckpt[1:, 0], ckpt.stride(0)      # V'(t) = v-plane of slot t + 1
        else:
            seed, sv_ld = v_out, n
        dX, dW, db = _layer_grads(ctx.layer, xb, wb, cur, ckpt, ctx.K, ctx.shape, ctx.x_requires_grad, seed,
                                  None, sv_ld=sv_ld, sv_scale=scale)
        return dX, dW, db, None


class HHLayer(torch.nn.Module):
    """Linear(n_in -> n_out, bf16 tcgen05) followed by n_out HH neurons per batch
    row, stepped over the leading time axis of x (T, B, n_in).

    Returns (V, spikes), both (T, B, n_out) fp32 on the device (outputs="v" or
    "spikes" keeps only that one -- the other comes back None and is never
    written); spikes carry
    gradients through the surrogate (seed_spike of adjoint.py:354-359), so
    layers stack.  HH parameters are fixed (like the reference's neuron in
    ReadoutModel); their gradients d_c_m / d_g_max of the last backward are in
    `param_grads` (device fp64 [1 + n_channels]).  budget=None keeps every
    state for the backward (the reference's full-storage mode), else
    checkpoints are spaced ceil(T/budget) (make_plan, adjoint.py:250-258).
    overlap_weight_grad=True computes dW / db on a side stream, overlapping the
    previous layer's BPTT in a stack; the grads land in .grad when the
    backward pass ends.  Limitation of that mode: autograd itself receives
    None for weight and bias, so torch.autograd.grad(loss, [weight]), tensor /
    module gradient hooks and DDP bucket hooks never see these gradients, and
    .grad is written even under autograd.grad -- use the default
    (overlap_weight_grad=False) with those APIs.

    proj selects the projection precision: "bf16" (default; config 4's bf16
    synaptic projection: x and W rounded to bf16, dI carried as bf16 hi + lo)
    or "bf16x3" (x, W and dI all split into bf16 hi + lo, three tensor-core
    products per GEMM: ~16 mantissa bits of every operand, the precision class
    of the reference's float64 DenseLayer, learn.py:210-211, at ~3x the
    projection FLOPs).
    """

    def __init__(self, n_in: int, n_out: int, params: HHParams | None = None, budget: int | None = None,
                 surrogate: SurrogateSpec | None = None, w_mean: float = 0.0, w_std: float | None = None,
                 check_finite: bool = True, device=None, outputs: str = "both",
                 overlap_weight_grad: bool = False, proj: str = "bf16"):
        super().__init__()
        if proj not in ("bf16", "bf16x3"):
            raise UsageError('proj must be "bf16" or "bf16x3"')
        self.proj = proj
        self.overlap_weight_grad = bool(overlap_weight_grad)
        if outputs not in ("both", "v", "spikes"):
            raise UsageError('outputs must be "both", "v" or "spikes"')
        self.outputs = outputs
        dev = device or D.require_cuda()
        p = params if params is not None else cortical_rs_params(dt=0.1)
        self.params = p.with_(dtype=np.float32)
        _table(self.params)
        self.budget = budget
        self.surrogate = surrogate if surrogate is not None else default_surrogate(self.params)
        std = w_std if w_std is not None else 1.0 / math.sqrt(n_in)
        self.weight = torch.nn.Parameter(torch.randn((n_out, n_in), device=dev) * std + w_mean)
        self.bias = torch.nn.Parameter(torch.zeros(n_out, device=dev))
        self.check_finite = check_finite
        self.param_grads = None
        self._rest = None

    def check(self):
        """Deferred form of check_finite (for check_finite=False training loops,
        which then never wait on the device inside a step): raise the
        NumericalOverflowError / GradientOverflowError of the last forward /
        backward, if any."""
        if getattr(self, "_last_bad", None) is not None:
            _raise_if_bad(self._last_bad)
        gb = getattr(self, "_last_gbad", None)
        if gb is not None and int(gb.item()) >= 0:
            raise GradientOverflowError("adjoint state became non-finite", int(gb.item()))

    def segment(self, T: int) -> int:
        return 1 if self.budget is None else make_plan(T, self.budget).segment_length

    def rest_state(self, n: int, dev):
        """Rest state (v_rest, steady-state gates) of n neurons; the forward only
        reads it, so one device copy per (n, device) is kept."""
        key = (n, str(dev))
        if self._rest is None or self._rest[0] != key:
            fr = steady_state_gates(self.params, self.params.v_rest)
            v = torch.full((n,), float(self.params.v_rest), dtype=torch.float32, device=dev)
            g = torch.empty((len(fr), n), dtype=torch.float32, device=dev)
            for i, f in enumerate(fr):
                g[i].fill_(f)
            self._rest = (key, v, g)
        return self._rest[1], self._rest[2]

    def forward(self, x: torch.Tensor):
        if x.dim() != 3:
            raise UsageError("HHLayer expects x of shape (T, B, n_in)")
        return _HHLayerFn.apply(x, self.weight, self.bias, self)

    def mse_loss(self, x: torch.Tensor, target: torch.Tensor | None = None) -> torch.Tensor:
        """MSE(V, target) of the layer's membrane trace (learn.py:80-88),
        differentiable into W, b and x.  target None (= 0) runs the fused
        kernels (_HHLayerMSEFn); otherwise learn.mse over the V output."""
        if x.dim() != 3:
            raise UsageError("HHLayer expects x of shape (T, B, n_in)")
        if target is None:
            return _HHLayerMSEFn.apply(x, self.weight, self.bias, self)
        from .learn import mse
        if self.outputs == "spikes":
            raise UsageError('mse_loss with a target needs the V output (outputs "both" or "v")')
        return mse(self(x)[0], target)


def allreduce_gradients(params, group=None, flat: torch.Tensor | None = None) -> torch.Tensor | None:
    """Data-parallel step of configs 3/4: average the gradients
    of `params` over the ranks of `group` with ONE all-reduce of a flat
    bucket (NCCL on the GPUs, gloo in the CPU tests), then copy the averages
    back.  flat: optional reusable bucket (float32, >= total numel).  Returns
    the bucket.  A no-op (None) without an initialised process group of
    more than one rank."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    grads = [p.grad for p in params if p.grad is not None]
    total = sum(g.numel() for g in grads)
    if flat is None or flat.numel() < total:
        flat = torch.empty(total, dtype=torch.float32, device=grads[0].device)
    off = 0
    for g in grads:
        flat[off:off + g.numel()].copy_(g.reshape(-1))
        off += g.numel()
    dist.all_reduce(flat[:total], group=group)
    flat[:total].div_(dist.get_world_size(group))
    off = 0
    for g in grads:
        g.copy_(flat[off:off + g.numel()].view_as(g))
        off += g.numel()
    return flat
