#!/usr/bin/env python
"""Throughput benchmark of the B200-native HH hot path (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...       (N > 1, one rank per GPU)

Metric (BASELINE.json): HH neuron-steps/s.  Workload at N = 1 is BASELINE
config 2: a 10,000,000-neuron population with the custom Na / K_dr / leak /
Ca_L / K_Ca channel set (6 gates, 5 channels, dt = 0.01 ms) driven by
I = 2 * Poisson(2) for 10,000 steps, fp32.  One "step" of this benchmark is
that whole simulation (1e11 neuron-steps): the device generates each
100-step chunk of stimulus (Philox) and the fused forward kernel advances the
population through it, writing the V trace and spike bitmap of the chunk
(4.0 GB + 125 MB per chunk, far above L2, so no flush is needed).  Weak
scaling: every rank owns its own 10M-neuron population (no collective on the
data path; independent neurons).

Extra keys: roofline (forward kernel vs the MUFU pipe peak measured live on
this GPU by hhb_pipe_probe), cpu_baseline (reference algorithm on the host
cores), e2e (the reference-facing `simulate` call with host numpy buffers),
fwd_bwd (forward + BPTT throughput on the config-3 shaped layer), clocks,
gpu_launches.  Only stdlib imports at module level: the CPU-baseline workers
are spawned processes that re-import this file.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
METRIC = "HH neuron-steps/sec (fwd; fwd+bwd) at 1/2/4/8 B200 vs CPU ref, % roofline"
UNIT = "neuron-steps/s"
# Transcendentals per neuron-step of the config-2 channel set in the
# reference's formulation (SURVEY.md §8 tau = 31: per gate 2 rate exps, 1 decay
# exp, 1/(a+b), plus 1 reciprocal per linoid/sigmoid rate).  The merged-form
# kernel evaluates the same step with fewer MUFU ops (shared rate exps, one
# reciprocal per gate); that count is read from the generated step itself.
# Algorithmic HBM bytes per neuron-step of the forward kernel: V write 4 +
# spike bit 1/8, plus the I read 4 when the stimulus is not fused.
TAU_C2 = 31
BYTES_PER_NS = 4.125
BYTES_PER_NS_UNFUSED = 8.125


def mufu_per_step(nat, params, which="fwd"):
    """MUFU ops (ex2 + rcp) per neuron-step of the generated regular-lane step
    (forward or backward), counted in the generated source; the ncu-measured
    XU instruction count of the same kernel is reported beside it."""
    src = nat.jit_source(params)
    # the paired (f32x2) merged step when generated: one ex2v / rcpv per neuron
    for head in (f"F2 step_{which}_m2(", f"float step_{which}_m(", f"float step_{which}_s("):
        if head in src:
            break
    body = src[src.index(head):]
    body = body[:body.index("\n}\n")]
    n = sum(body.count(k) for k in ("ex2f_(", "rcpf_(", "ex2v<H>(", "rcpv<H>("))
    return n, head.split()[1][:-1]


def load_json(*parts):
    path = os.path.join(ROOT, *parts)
    try:
        with open(path) as f:
            return json.load(f)
    except (OSError, ValueError):
        return {}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def layer_kernels(torch, step, reps=7):
    """Per-component kernel times of an HH-layer training step, from CUDA
    events recorded on each component's own stream (layer.TIMERS) around its
    launches, over `reps` eager steps; the median step is kept per component
    (a GPU spin before each start event hides the host's launch preparation,
    which an occasional allocation can still outlast):
    {name: {ms_per_step, launches_per_step, units_per_s}}."""
    from paper_2601_21407_b200 import layer as L
    torch.cuda.synchronize()
    L.TIMERS = {}
    try:
        for _ in range(reps):
            step()
        torch.cuda.synchronize()
        recs = L.TIMERS
    finally:
        L.TIMERS = None
    out = {}
    for name, rr in recs.items():
        per = len(rr) // reps
        steps = [rr[k * per:(k + 1) * per] for k in range(reps)]
        ms_units = sorted((sum(a.elapsed_time(b) for a, b, _ in st), sum(u for _, _, u in st)) for st in steps)
        ms, units = ms_units[reps // 2]
        out[name] = {"ms_per_step": ms, "launches_per_step": per,
                     "units_per_s": units / (ms * 1e-3) if ms > 0 else None}
    return out


# reference-formulation transcendentals per neuron-step of the RS set (SURVEY
# §8 d7): forward tau_f = 16; backward with reuse tau_b = tau_f + 2 = 18
TAU_RS_F, TAU_RS_B = 16, 18


def layer_roofline(nat, params, kern, step_ms, mufu_peak, dual_grads=True, proj_products=1):
    """Roofline of an HH-layer training step: the dominant kernel (the BPTT
    kernel hh_bwd2) against the live MUFU peak, with the forward kernel and the
    projection GEMM beside it (GEMM against MEASURED_PEAKS bf16_tflops)."""
    peaks = load_json("MEASURED_PEAKS.json")
    prof = load_json("profiles", "k_bptt.json")
    mb, fnb = mufu_per_step(nat, params, "bwd")
    mf, fnf = mufu_per_step(nat, params, "fwd")
    b, f, g = kern.get("hh_bptt", {}), kern.get("hh_forward", {}), kern.get("proj_gemm", {})
    bw = b.get("units_per_s") or 0.0
    fw = f.get("units_per_s") or 0.0
    roof = {"bound": "sfu", "kernel": "hh_bwd2 (NVRTC-specialised merged-form BPTT, hhb_backward)",
            "achieved": mb * bw / 1e9, "peak": mufu_peak / 1e9, "unit": "Gop/s", "frac": mb * bw / mufu_peak,
            "traffic": prof.get("dram_bytes_per_neuron_step"),
            "algorithmic": f"{mb} MUFU ops per neuron-step ({fnb}, counted in the generated source) x "
                           "neuron-steps per launch",
            "peak_source": "measured live: hhb_pipe_probe MUFU.EX2 throughput on this GPU",
            "avg_launch_ms": b.get("ms_per_step", 0) / max(1e-9, b.get("launches_per_step", 1)),
            "share_of_step": b.get("ms_per_step", 0) / step_ms,
            "neuron_steps_per_s": bw,
            "reference_tau": {"transcendentals_per_neuron_step": TAU_RS_B, "frac": TAU_RS_B * bw / mufu_peak},
            "forward_kernel": {"kernel": "hh_fwd_v4 (training forward, checkpoints)", "mufu_per_neuron_step": mf,
                               "neuron_steps_per_s": fw, "frac": mf * fw / mufu_peak,
                               "reference_tau_frac": TAU_RS_F * fw / mufu_peak,
                               "share_of_step": f.get("ms_per_step", 0) / step_ms},
            "kernels_ms_per_step": {k: v["ms_per_step"] for k, v in kern.items()}}
    if "inst_per_neuron_step" in prof and bw:
        # instruction-issue view (4 warp-instructions / clk / SM = 128 thread-instructions):
        # the bound that binds this kernel (ncu: issue active 78 %, MUFU 39 %, FMA 47 %)
        sm_hz = 1965.0e6
        issue_bound = 148 * 128 * sm_hz / prof["inst_per_neuron_step"]
        roof["issue"] = {"inst_per_neuron_step": prof["inst_per_neuron_step"],
                         "bound_neuron_steps_per_s": issue_bound, "frac": bw / issue_bound,
                         "source": prof.get("source")}
    if "xu_inst_per_neuron_step" in prof:
        roof["mufu_check"] = {"source_count": mb, "ncu_sass_count": prof["xu_inst_per_neuron_step"],
                              "agree": abs(prof["xu_inst_per_neuron_step"] - mb) <= 0.05 * mb}
        roof["ncu"] = {k: prof[k] for k in ("xu_inst_per_neuron_step", "inst_per_neuron_step", "issue_active_pct",
                                            "xu_pipe_pct", "fma_pipe_pct", "source") if k in prof}
    if g.get("units_per_s"):
        pk = peaks.get("bf16_tflops", 1648.7)
        # tensor work issued: the bf16x3 projection runs three products per
        # algorithmic MAC (x_hi.W_hi + x_lo.W_hi + x_hi.W_lo)
        roof["gemm"] = {"kernel": ("k_umma_gemm_2sm_cvt (tcgen05 cta_group::2, x converted and hi/lo-split on chip, "
                                   "three products)" if proj_products == 3 else
                                   "k_umma_gemm_2sm (tcgen05 cta_group::2, projection x W^T)"),
                        "achieved_tflops": proj_products * g["units_per_s"] / 1e12, "peak_tflops": pk,
                        "frac": proj_products * g["units_per_s"] / 1e12 / pk,
                        "algorithmic_tflops": g["units_per_s"] / 1e12, "products_per_mac": proj_products,
                        "peak_source": "MEASURED_PEAKS.json bf16_tflops" if "bf16_tflops" in peaks else "fallback",
                        "share_of_step": g.get("ms_per_step", 0) / step_ms}
        for name in ("grad_w", "grad_x"):
            if kern.get(name, {}).get("units_per_s"):
                roof["gemm"][name + "_tflops_algorithmic"] = kern[name]["units_per_s"] / 1e12
        if dual_grads:
            roof["gemm"]["note"] = ("gradient GEMMs carry dI as bf16 hi + lo (two tensor-core products per "
                                    "algorithmic MAC): their algorithmic TFLOP/s is half the tensor work rate")
    return roof


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--neurons", type=int, default=10_000_000)
    ap.add_argument("--sim-steps", type=int, default=10_000)
    ap.add_argument("--chunk", type=int, default=500)   # steps per launch (V trace buffer 20 GB at 10M neurons)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / fwd_bwd / cpu legs")
    ap.add_argument("--no-fuse", action="store_true", help="stimulus as a separate kernel + HBM buffer")
    ap.add_argument("--legs", default="", help="comma-separated subset of the secondary legs (default: all)")
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl",
                    help="torch.distributed backend under torchrun (gloo: a smoke of the N > 1 code path, "
                         "ranks may share one GPU)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def c2_params(dtype):
    sys.path.insert(0, ROOT)
    from paper_2601_21407_b200.defaults import na_kdr_cal_kca_params
    return na_kdr_cal_kca_params(dt=0.01).with_(dtype=dtype)


# --------------------------------------------------------------------------- clocks
class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, val in zip(names, f[5:9]):
                if val.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------------------- CPU legs
def cpu_leg(seconds, n_total, dtype="float32"):
    sys.path.insert(0, ROOT)
    from oracle import cpu_baseline
    from paper_2601_21407_b200.defaults import na_kdr_cal_kca_params
    pdict = na_kdr_cal_kca_params(dt=0.01).to_dict()
    return cpu_baseline.run(pdict, dtype=dtype, n_total=n_total, seconds=seconds)


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    secs = max(2.0, args.cpu_seconds / 2)
    for _ in range(args.warmup):
        cpu_leg(min(secs, 2.0), 1 << 21)
    tot_ns, tot_s, last = 0, 0.0, None
    for _ in range(args.steps):
        r = cpu_leg(secs, 1 << 21)
        tot_ns += r["neuron_steps"]
        tot_s += r["seconds"]
        last = r
    value = tot_ns / tot_s
    sample = (f"reference hh_step loop (oracle port, fp32 mode) on {last['cores']} processes x "
              f"{last['n_local']} neurons of the config-2 population, ~{secs:.0f} s per step")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": config_dict(args),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": last["cores"], "kind": "port",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def config_dict(args):
    return {"workload": "BASELINE config 2: HH population, custom Na/K_dr/leak/Ca_L/K_Ca channels "
                        "(6 gates), I = 2*Poisson(2), fp32 forward, V + spike trace recorded",
            "neurons_per_gpu": args.neurons, "sim_steps": args.sim_steps, "dt_ms": 0.01,
            "chunk_steps": args.chunk, "parallelism": f"neuron-shard x{args.gpus} (weak, no collective)",
            "l2": f"outputs per chunk ({args.neurons * args.chunk * 4 / 1e9:.0f} GB V trace) exceed the 126 MB L2; "
                  "no flush needed"}


# --------------------------------------------------------------------------- GPU legs
def probe_mufu_peak(torch, nat, dev):
    """MUFU ex2 throughput of this GPU, ops/s (live roofline denominator)."""
    import ctypes as C
    sink = torch.zeros(1, device=dev)
    ops = C.c_int64(0)
    lib = nat.load()
    for _ in range(2):
        nat.check(lib.hhb_pipe_probe(0, 2000, sink.data_ptr(), C.byref(ops), None), "probe")
    torch.cuda.synchronize()
    best = 0.0
    for which in (0, 2):
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            nat.check(lib.hhb_pipe_probe(which, 20000, sink.data_ptr(), C.byref(ops),
                                         torch.cuda.current_stream().cuda_stream), "probe")
            e1.record()
            e1.synchronize()
            best = max(best, ops.value / (e0.elapsed_time(e1) * 1e-3)) if which == 0 else best
    return best


def e2e_leg(torch, args, params, rank):
    """Reference-facing call with host buffers: dynamics.simulate(numpy) on the
    full population for a bounded number of steps (H2D of I, D2H of the
    float64 V trace and bool spikes inside the timed region)."""
    import numpy as np
    from paper_2601_21407_b200 import dynamics as Dy
    from paper_2601_21407_b200._pipeline import pinned_empty
    n, T = args.neurons, args.e2e_steps
    rng = np.random.default_rng(rank)
    # the step's inputs live in pinned host memory (the e2e contract); simulate
    # DMAs them as they are
    i_host = pinned_empty((T, n), np.float32)
    i_host[...] = 2.0 * rng.poisson(2.0, size=(T, n))
    tr = Dy.simulate(params, i_host)           # warm-up: module, device + pinned-host caches
    h2d = i_host.nbytes
    d2h = tr.v_series.nbytes + tr.spike_series.nbytes
    del tr                                     # a caller loop drops the previous Trace
    torch.cuda.synchronize()
    reps = 3
    el = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        tr = Dy.simulate(params, i_host)
        torch.cuda.synchronize()
        el += time.perf_counter() - t0
        del tr
    el /= reps
    return {"value": n * T / el, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "seconds_per_step": el,
            "sample": f"simulate(numpy float32 I[{T}, {n}], pinned) -> Trace(float64 V, bool spikes)"}


def graph_step(torch, step):
    """Capture one training step into a CUDA graph (after eager warm-up: JIT
    modules, workspaces and the gradient tensors exist).  None if capture fails."""
    try:
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            step()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        torch.cuda.synchronize()
        return g
    except Exception as e:  # noqa: BLE001 -- fall back to eager timing
        print(f"bench: CUDA graph capture failed ({e}); timing eager steps", file=sys.stderr)
        return None


def cpu_layers_leg(sizes, seconds):
    """Same-run CPU baseline of configs 3 / 4: the reference composition
    (DenseLayer -> simulate -> backward_through_time -> dW einsum, oracle port)
    on every host core, one batch-1 shard per process."""
    sys.path.insert(0, ROOT)
    from oracle import cpu_baseline
    from paper_2601_21407_b200.defaults import cortical_rs_params
    r = cpu_baseline.run_layers(cortical_rs_params(dt=0.1).to_dict(), sizes, 100, seconds=seconds)
    return {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port", "cpu_model": cpu_model(),
            "sample": f"reference composition (oracle port of learn.py:238-274 + adjoint.py:281-365, float64) "
                      f"{'->'.join(map(str, sizes))} x 100 steps, {r['samples']} batch-1 samples on "
                      f"{r['cores']} processes in {r['seconds']:.1f} s"}


def fwd_bwd_leg(torch, dev, proj="bf16", mufu_peak=None, cpu_seconds=0.0):
    """BASELINE config 3: differentiable HH SNN layer forward + BPTT, batch 256,
    784 -> 1024 RS neurons, 100 steps, x = Bernoulli(0.2) + 0.1 N(0,1),
    W ~ N(0.05, 0.1^2), loss MSE(V, 0).  One step = tcgen05 projection (bf16,
    or bf16x3: the fp32-class split that meets the gradient contract against
    the reference's float64 operands), HH forward (full storage), BPTT,
    dW / db gradient GEMMs.  x is the data: no input gradient, as the
    reference's first layer (SURVEY §8 d3 lists the forward and dW GEMMs; the
    CPU composition, oracle/cpu_baseline.py, computes none either)."""
    from paper_2601_21407_b200 import _native as nat
    from paper_2601_21407_b200.layer import HHLayer
    B, N, T, K_in = 256, 1024, 100, 784
    torch.manual_seed(0)
    # HHB_BENCH_C3_OVERLAP=1: dW / db on a side stream (they overlapped dX when
    # the leg also produced the input gradient)
    ov = os.environ.get("HHB_BENCH_C3_OVERLAP", "0") not in ("", "0")
    layer = HHLayer(K_in, N, w_mean=0.05, w_std=0.1, check_finite=False, device=dev, proj=proj,
                    overlap_weight_grad=ov)
    g = torch.Generator(device=dev).manual_seed(0)
    x = ((torch.rand((T, B, K_in), device=dev, generator=g) < 0.2).float()
         + 0.1 * torch.randn((T, B, K_in), device=dev, generator=g))

    def step():
        layer.zero_grad(set_to_none=True)
        # MSE(V, 0) fused into the HH kernels: sum V^2 accumulated by the
        # forward, the seed 2 V / numel (learn.py:86-88) read from the
        # checkpoints by the BPTT kernel -- no V trace written, no seed pass
        layer.mse_loss(x).backward()

    def timed(fn, reps=10):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    for _ in range(3):
        step()
    eager_ms = timed(step)
    # the whole training step (forward, loss, backward: ~25 launches) as one
    # CUDA graph: the same kernels without the host launch gaps
    graph = graph_step(torch, step)
    ms = timed(graph.replay) if graph is not None else eager_ms
    layer.check()      # the overflow checks, deferred out of the timed steps
    out = {"value": B * N * T / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "eager_ms_per_step": eager_ms,
           "cuda_graph": graph is not None, "proj": proj,
           "config": f"BASELINE config 3: HH SNN layer 784->1024, batch 256, 100 steps, {proj} tcgen05 "
                     + ("projection (fp32 x rounded and hi/lo-split on chip inside the GEMM) " if proj == "bf16x3"
                        else "projection ") +
                     "+ fp32 HH forward + full-storage BPTT + bf16 hi/lo weight-gradient "
                     "GEMM (x is the data: no input gradient, as the reference's first layer), "
                     "loss MSE(V, 0) fused into the HH kernels (layer.mse_loss; one unit = one "
                     "neuron-step through forward and backward)",
           "parity": ("dW within 1e-4 of the float64 reference on the UNROUNDED operands "
                      "(profiles/r2_parity_c3_unrounded.md)" if proj == "bf16x3" else
                      "within 3e-5 of the float64 reference on bf16-rounded operands, 3-4e-3 on the "
                      "unrounded ones (profiles/r2_parity_c3_unrounded.md)")}
    if mufu_peak:
        out["roofline"] = layer_roofline(nat, layer.params, layer_kernels(torch, step), ms, mufu_peak,
                                         proj_products=3 if proj == "bf16x3" else 1)
    if cpu_seconds > 0:
        out["cpu_baseline"] = cpu_layers_leg([784, 1024], cpu_seconds)
    return out


def c5_leg(torch, dev, steps=1000, with_cpu=False, scale=0.5):
    """BASELINE config 5: recurrent HH cortex, build_network(scale=0.5, seed=0)
    (38,586 RS neurons, 71.2M synapses, delays up to 193 steps), REST_CONFIG,
    fp32, device Philox background; per step: ring drain + PSP + background,
    HH step, spike bitmap (all-gathered over NCCL when N > 1), fixed-point
    delivery -- on one GPU all steps in one persistent cooperative kernel.
    One unit = one neuron-step of the whole network (strong scaling)."""
    import numpy as np
    import torch.distributed as dist
    from paper_2601_21407_b200 import network as N
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    t0 = time.perf_counter()
    topo = N.build_network(scale, 0)
    build_s = time.perf_counter() - t0
    ex, ex_kind = None, None
    if world > 1:
        if dist.get_backend() == "nccl" and os.environ.get("HHB_BENCH_C5_EXCHANGE", "library") == "library":
            # the library exchange (hhb_spk_step: ncclAllGather + delivery), captured into
            # the 64-step CUDA graphs with the step kernels; a hung or failed peer
            # surfaces as ExchangeError after 120 s (the communicator is aborted)
            ex = N.LibraryExchange(topo.n_neurons, timeout_s=120.0)
            ex_kind = "library ncclAllGather in CUDA graphs"
        elif dist.get_backend() == "nccl":
            ex, ex_kind = N.allgather_exchange(topo.n_neurons), "torch.distributed all-gather (NCCL, eager)"
        else:
            ex, ex_kind = N.allgather_exchange(topo.n_neurons), "torch.distributed all-gather (gloo, host-staged)"
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=dev, dtype=np.float32, rank=rank, world=world,
                          exchange=ex, background="philox", seed=1)
    graphs = world == 1 or isinstance(ex, N.LibraryExchange)
    for _ in range(100):
        net.step()
    if graphs:
        net.advance(128)         # capture + warm the graph
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    if graphs:
        net.advance(steps, wait=False)   # one persistent cooperative kernel (graph replay if unavailable)
    else:
        for _ in range(steps):
            net.step()
    e1.record()
    if hasattr(ex, "wait"):
        ex.wait()                # NCCL error / timeout check, outside the timed events
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    m = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(m, op=dist.ReduceOp.MAX)
    ms = float(m.item())
    extra = {}
    if with_cpu:
        # same-run CPU baseline: the reference's step_network (oracle port) on one core
        # (network stepping is serial in the reference), 100 warm-up + 200 timed steps
        sys.path.insert(0, ROOT)
        from oracle import cpu_baseline
        cfg = N.REST_CONFIG
        r = cpu_baseline.run_network(cfg.resolved_neuron().to_dict(), topo.syn_offsets, topo.syn_target,
                                     topo.syn_weight, topo.syn_delay, topo.max_delay,
                                     N.background_lambda(topo, N.make_background(cfg), cfg.dt), cfg.bg_mean,
                                     cfg.bg_std, float(np.exp(-cfg.dt / cfg.psp_tau_ms)), steps=200, warm=100)
        extra["cpu_baseline"] = {"value": r["value"], "unit": UNIT, "cores": 1, "kind": "port",
                                 "cpu_model": cpu_model(), "ms_per_network_step": 1e3 * r["seconds"] / r["steps"],
                                 "sample": "reference step_network (oracle port of cortex.py:273-310, float64, "
                                           "numpy compound-Poisson background) on one core, steps 100-299 "
                                           f"({r['spikes_per_step']:.1f} spikes / step)"}
    return {"value": topo.n_neurons * steps / (ms * 1e-3), "unit": UNIT, "ms_per_network_step": ms / steps, **extra,
            "steps": steps, "neurons": topo.n_neurons, "synapses": topo.n_synapses,
            "host_build_s": build_s,
            "path": ("persistent kernel" if net.persistent_ok() and not getattr(net, "_no_persist", False)
                     else "cuda graphs of 64 steps") + (f" + {ex_kind}" if ex_kind else "") if graphs
            else f"eager steps + {ex_kind}",
            "config": f"BASELINE config 5: recurrent HH cortex scale {scale} ({topo.n_neurons:,} neurons, "
                      f"{topo.n_synapses / 1e6:.1f}M synapses), REST_CONFIG, fp32, device Philox background"}


def c1_leg(torch, dev, with_cpu=True):
    """BASELINE config 1 (the reference's CPU-runnable case): squid axon
    Na/K/leak, 1,024 neurons x 10,000 steps, dt 0.01 ms, constant 10 uA/cm^2,
    fp32 forward, V + spikes recorded.  One fused launch; latency-bound (one
    wave of 256 threads walks 10,000 dependent steps), so reported as an
    absolute rate, not a roofline fraction.  Beside it the oracle port of the
    reference loop on one host core over the full config (test/bench
    infrastructure only) and the reference-facing numpy call."""
    import numpy as np
    from paper_2601_21407_b200 import dynamics as Dy
    from paper_2601_21407_b200.defaults import squid_axon_params
    p = squid_axon_params(dt=0.01).with_(dtype=np.float32)
    n, T = 1024, 10000
    i = torch.full((T, n), 10.0, dtype=torch.float32, device=dev)
    for _ in range(2):
        tr = Dy.simulate(p, i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        tr = Dy.simulate(p, i)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    spikes = int(tr.spike_series[:, 0].sum().item())
    i_host = np.full((T, n), 10.0, dtype=np.float32)
    Dy.simulate(p, i_host)
    calls = []
    for _ in range(9):             # median of 9 host-buffer calls (one call is noisy)
        t0 = time.perf_counter()
        Dy.simulate(p, i_host)
        calls.append(time.perf_counter() - t0)
    e2e_s = sorted(calls)[len(calls) // 2]
    out = {"value": n * T / (ms * 1e-3), "unit": UNIT, "ms_per_run": ms, "spikes_per_neuron": spikes,
           "e2e_numpy": {"value": n * T / e2e_s, "seconds": e2e_s, "seconds_min": min(calls),
                         "sample": "simulate(numpy float32 I[10000, 1024]) -> Trace(float64 V, bool spikes)"},
           "config": "BASELINE config 1: squid axon, 1,024 neurons x 10,000 steps, I = 10 uA/cm^2, fp32"}
    if with_cpu:
        sys.path.insert(0, ROOT)
        from oracle import hh_oracle as O
        p32 = squid_axon_params(dt=0.01).with_(dtype=np.float32)
        t0 = time.perf_counter()
        O.simulate(p32, i_host, dtype=np.float32)
        cs = time.perf_counter() - t0
        out["cpu_oracle"] = {"value": n * T / cs, "seconds": cs, "cores": 1, "kind": "port",
                             "sample": "the whole config on one host core (oracle port of the reference loop, fp32)"}
    return out


def morph_leg(torch, dev):
    """multicompartment neurons (morphology.py mirror over
    hhb_morph_forward): the coincidence-detection graph (active squid soma +
    3 two-compartment passive dendrites, 7 compartments, 6 axial edges) for a
    batch of 262,144 independent neurons x 400 steps, fp32, random pulse
    currents.  One unit = one compartment-step."""
    import numpy as np
    from paper_2601_21407_b200 import morphology as M
    from paper_2601_21407_b200.defaults import squid_axon_params
    soma = squid_axon_params().with_(dtype=np.float32)
    dend = M.passive_params(dt=soma.dt).with_(dtype=np.float32)
    comps = {"soma": soma}
    edges = []
    for d in (1, 2, 3):
        comps[f"d{d}p"], comps[f"d{d}d"] = dend, dend
        edges += [M.Edge("soma", f"d{d}p", M.DEMO_G_AXIAL), M.Edge(f"d{d}p", f"d{d}d", M.DEMO_G_AXIAL)]
    graph = M.CompartmentGraph(comps, edges, "soma")
    B, T = 262144, 400
    g = torch.Generator(device=dev).manual_seed(0)
    i = (torch.rand((T, 7, B), device=dev, generator=g) < 0.05).float() * 36.0
    for _ in range(3):
        M.simulate_morphology(graph, i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 3
    tr = None
    for _ in range(reps):
        tr = None                 # one output set alive at a time: the allocator reuses its blocks
        tr = M.simulate_morphology(graph, i)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return {"value": 7 * B * T / (ms * 1e-3), "unit": "compartment-steps/s", "ms_per_step": ms,
            "spikes": int(tr.spike_series[:, 0].sum().item()),
            "config": "coincidence graph (7 compartments, 2 channel tables, 6 axial edges) x 262,144 neurons "
                      "x 400 steps, fp32, V trace + spikes recorded (one unit = one compartment-step)"}


def c5_replicas_leg(torch, dev, topo=None, replicas=(8, 32, 64), steps=640):
    """Config 5 in the paper's "replicas x speed" view: R
    independent copies of the scale-0.5 network stepped together on one GPU
    (CortexReplicas: one input, one HH and one delivery launch per step for all
    replicas, CUDA-graph replay).  One unit = one neuron-step of one replica."""
    import numpy as np
    from paper_2601_21407_b200 import network as N
    topo = topo or N.build_network(0.5, 0)
    out = {}
    for R in replicas:
        rep = N.CortexReplicas(topo, N.REST_CONFIG, R, device=dev, dtype=np.float32, seed=1)
        rep.advance(128)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rep.advance(steps)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out[str(R)] = {"ms_per_network_step": ms, "value": R * topo.n_neurons / (ms * 1e-3)}
        del rep
        torch.cuda.empty_cache()
    best = max(out, key=lambda k: out[k]["value"])
    return {"value": out[best]["value"], "unit": UNIT, "replicas": int(best), "by_replicas": out,
            "config": "BASELINE config 5 network (scale 0.5, 38,586 neurons, 71.2M synapses), R independent "
                      "replicas per GPU, fp32, device background (one unit = one neuron-step of one replica)"}


def c4_leg(torch, dev, mufu_peak=None, cpu_seconds=0.0):
    """BASELINE config 4: stacked HH SNN 784 -> 2048 -> 2048 -> 10 (RS neurons),
    batch 256, 100 steps, cross-entropy on the time-mean output V, Adam; one
    training step per unit of work."""
    from paper_2601_21407_b200.layer import HHLayer, allreduce_gradients
    B, T = 256, 100
    torch.manual_seed(1)
    # hidden layers hand on spikes only, the readout layer V only: the unused
    # trace of each layer is never written.  Weights: every layer spikes (~1.5
    # spikes per neuron in layer 1, ~1 in layers 2 and 3 over the 100 steps,
    # checked with the oracle); W ~ N(0.02, 0.05^2) above layer 1 left layers
    # 2 and 3 silent
    # (weight gradients on a side stream overlap the next-lower layer's BPTT)
    ov = os.environ.get("HHB_BENCH_NO_OVERLAP", "0") in ("", "0")
    net = torch.nn.ModuleList([
        HHLayer(784, 2048, w_mean=0.05, w_std=0.1, check_finite=False, device=dev, outputs="spikes",
                overlap_weight_grad=ov),
        HHLayer(2048, 2048, w_mean=0.3, w_std=0.1, check_finite=False, device=dev, outputs="spikes",
                overlap_weight_grad=ov),
        HHLayer(2048, 10, w_mean=0.3, w_std=0.1, check_finite=False, device=dev, outputs="v",
                overlap_weight_grad=ov)])
    import torch.distributed as dist
    world = dist.get_world_size() if dist.is_initialized() else 1
    # capturable Adam keeps its step counters on the device (CUDA-graph safe)
    opt = torch.optim.Adam(net.parameters(), lr=5e-4, capturable=(world == 1), fused=True)
    g = torch.Generator(device=dev).manual_seed(1)
    x = (torch.rand((T, B, 784), device=dev, generator=g) < 0.2).float() \
        + 0.1 * torch.randn((T, B, 784), device=dev, generator=g)
    y = torch.randint(0, 10, (B,), device=dev, generator=g)
    params = [p for p in net.parameters()]
    flat = torch.empty(sum(p.numel() for p in params), dtype=torch.float32, device=dev) if world > 1 else None

    def step():
        opt.zero_grad(set_to_none=True)
        h = x
        for lyr in net[:-1]:
            _, h = lyr(h)
        v, _ = net[-1](h)
        loss = torch.nn.functional.cross_entropy(v.mean(0), y)
        loss.backward()
        if world > 1:  # data parallel over the batch shards of the ranks
            allreduce_gradients(params, flat=flat)
        opt.step()
        return loss.detach()     # no autograd graph kept alive across steps (graph capture)

    def timed(fn, reps=5):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) / reps

    for _ in range(3):
        loss = step()
    eager_ms = timed(step)
    # one CUDA graph per training step (forward, CE, backward, Adam) on one GPU;
    # under torchrun the NCCL all-reduce keeps the step eager
    box = {}
    graph = graph_step(torch, lambda: box.__setitem__("loss", step())) if world == 1 else None
    ms = timed(graph.replay) if graph is not None else eager_ms
    if graph is not None:
        loss = box["loss"]
    for lyr in net:
        lyr.check()
    ns = B * T * (2048 + 2048 + 10)
    extra = {}
    if mufu_peak:
        from paper_2601_21407_b200 import _native as nat
        extra["roofline"] = layer_roofline(nat, net[0].params, layer_kernels(torch, step), ms, mufu_peak)
    if cpu_seconds > 0:
        extra["cpu_baseline"] = cpu_layers_leg([784, 2048, 2048, 10], cpu_seconds)
    return {"value": ns / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "eager_ms_per_step": eager_ms,
            "cuda_graph": graph is not None, "loss": float(loss.item()), **extra,
            "config": "BASELINE config 4: stacked HH SNN 784->2048->2048->10, batch 256, 100 steps, "
                      "bf16 tcgen05 projections, fp32 gating state, CE on time-mean V, Adam "
                      "(one unit = one neuron-step through forward and backward)"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    rank, world, local = dist_env()
    import numpy as np
    import torch
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    from paper_2601_21407_b200 import _native as nat
    from paper_2601_21407_b200.population import Population, PoissonCurrent

    local = local % torch.cuda.device_count()        # gloo smoke: ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import datetime
        # a dead or hung rank fails the collective after 10 min instead of hanging the job
        tmo = datetime.timedelta(minutes=10)
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=dev, timeout=tmo)
        else:
            dist.init_process_group("gloo", timeout=tmo)
    nat.load()

    params = c2_params(np.float32)
    pop = Population(params, args.neurons, chunk=args.chunk, device=dev, neuron_base=rank * args.neurons,
                     fuse_stimulus=not args.no_fuse)
    stim = PoissonCurrent(2.0, 2.0, seed=1234)

    # warm-up: W full passes
    for _ in range(args.warmup):
        pop.reset()
        pop.advance(stim, args.sim_steps)
    torch.cuda.synchronize()

    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    events = []
    step_ev = []
    launches0 = pop.launches
    for _ in range(args.steps):
        pop.reset()
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        pop.advance(stim, args.sim_steps, events=events)
        s1.record()
        step_ev.append((s0, s1))
    torch.cuda.synchronize()
    launches = pop.launches - launches0
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    from paper_2601_21407_b200.dynamics import _raise_if_bad
    _raise_if_bad(pop.first_bad)
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    total_ms = sum(step_ms)
    fwd_ms = sum(e1.elapsed_time(e2) for _, e1, e2 in events)
    stim_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in events)
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())

    ns_per_rank = args.neurons * args.sim_steps * args.steps
    value = ns_per_rank * world / (total_ms * 1e-3)

    # roofline of the dominant kernel (hhb_forward), from its own events
    n_fwd = len(events)
    fwd_avg_s = fwd_ms * 1e-3 / n_fwd
    ns_per_launch = args.neurons * args.chunk
    mufu_peak = probe_mufu_peak(torch, nat, dev)
    mufu, step_fn = mufu_per_step(nat, params)
    bpn = BYTES_PER_NS_UNFUSED if args.no_fuse else BYTES_PER_NS
    achieved = mufu * ns_per_launch / fwd_avg_s
    prof = {}
    tp = os.path.join(ROOT, "profiles", "k_forward_dram.json")
    if os.path.exists(tp):
        try:
            prof = json.load(open(tp))
        except (OSError, ValueError):
            prof = {}
    traffic = prof["bytes_per_neuron_step"] * ns_per_launch if "bytes_per_neuron_step" in prof else None
    peaks = {}
    pk = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(pk):
        peaks = json.load(open(pk))
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    kname = ("hh_fwdp_v4" if not args.no_fuse else "hh_fwd_v4") + " (NVRTC-specialised, hhb_forward"
    kname += "_poisson)" if not args.no_fuse else ")"
    roof = {"bound": "sfu", "achieved": achieved / 1e9, "peak": mufu_peak / 1e9, "unit": "Gop/s",
            "frac": achieved / mufu_peak, "traffic": traffic, "kernel": kname,
            "algorithmic": f"{mufu} MUFU ops per neuron-step ({step_fn}: shared rate exps + one "
                           f"reciprocal per gate) x {ns_per_launch} neuron-steps per launch",
            "peak_source": "measured live: hhb_pipe_probe MUFU.EX2 throughput on this GPU",
            "avg_launch_ms": fwd_avg_s * 1e3, "share_of_step": fwd_ms / sum(step_ms),
            "reference_tau": {"transcendentals_per_neuron_step": TAU_C2,
                              "frac": TAU_C2 * ns_per_launch / fwd_avg_s / mufu_peak,
                              "note": "the reference formulation's 31 transcendentals per neuron-step "
                                      "delivered per second, over the same MUFU peak"},
            "hbm": {"achieved_gbs": bpn * ns_per_launch / fwd_avg_s / 1e9,
                    "peak_gbs": hbm_peak, "frac": bpn * ns_per_launch / fwd_avg_s / 1e9 / hbm_peak,
                    "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback"}}
    if "xu_inst_per_neuron_step" in prof and not args.no_fuse:
        # the numerator's MUFU count (generated source) against the executed MUFU
        # instructions per neuron-step of an ncu capture of the same kernel
        roof["mufu_check"] = {"source_count": mufu, "ncu_sass_count": prof["xu_inst_per_neuron_step"],
                              "agree": abs(prof["xu_inst_per_neuron_step"] - mufu) <= 0.05 * mufu}
    if "inst_per_neuron_step" in prof and not args.no_fuse:
        # instruction-issue view: 4 warp-instructions / clk / SM = 128 thread-instructions
        sm_hz = (clk.get("sm_mhz") or 1965.0) * 1e6
        issue_bound = 148 * 128 * sm_hz / prof["inst_per_neuron_step"]
        roof["issue"] = {"inst_per_neuron_step": prof["inst_per_neuron_step"],
                         "bound_neuron_steps_per_s": issue_bound,
                         "frac": ns_per_launch / fwd_avg_s / issue_bound,
                         "source": prof.get("source")}

    extras = {}

    only = set(args.legs.split(",")) if args.legs else None

    def leg(name, fn):
        if only is not None and name not in only:
            return
        # a failing secondary leg is reported in the line, not fatal to it;
        # each leg starts from an emptied allocator cache (the previous legs'
        # graph pools and temporaries would otherwise make its first
        # allocations pay for fragmentation)
        import gc
        gc.collect()
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        try:
            extras[name] = fn()
        except Exception as e:  # noqa: BLE001
            extras[name] = {"error": f"{type(e).__name__}: {e}"[:300]}
            print(f"bench: {name} failed: {e}", file=sys.stderr)

    if not args.no_extras:
        leg("e2e", lambda: e2e_leg(torch, args, params, rank))
        if "seconds_per_step" in extras.get("e2e", {}):
            ev = torch.tensor([extras["e2e"]["seconds_per_step"]], dtype=torch.float64, device=dev)
            if world > 1:
                dist.all_reduce(ev, op=dist.ReduceOp.MAX)
            extras["e2e"]["value"] = args.neurons * args.e2e_steps * world / float(ev.item())
        cpu_ok = rank == 0 and world == 1 and not args.no_cpu
        leg("fwd_bwd", lambda: fwd_bwd_leg(torch, dev, "bf16x3", mufu_peak, args.cpu_seconds if cpu_ok else 0.0))
        leg("fwd_bwd_bf16", lambda: fwd_bwd_leg(torch, dev, "bf16", mufu_peak))
        leg("c1", lambda: c1_leg(torch, dev, with_cpu=(rank == 0)))
        leg("c4_train_step", lambda: c4_leg(torch, dev, mufu_peak, args.cpu_seconds if cpu_ok else 0.0))
        leg("c5_network", lambda: c5_leg(torch, dev, with_cpu=cpu_ok))
        leg("c5_network_100m", lambda: c5_leg(torch, dev, scale=0.59))
        leg("morphology", lambda: morph_leg(torch, dev))
        leg("c5_replicas", lambda: c5_replicas_leg(torch, dev))
        # data parallel (weak: batch 256 per rank): whole-job rate over the slowest rank
        for name, ns in (("fwd_bwd", 256 * 1024 * 100), ("fwd_bwd_bf16", 256 * 1024 * 100),
                         ("c4_train_step", 256 * 100 * (2048 + 2048 + 10))):
            if world > 1 and "ms_per_step" in extras.get(name, {}):
                fb = torch.tensor([extras[name]["ms_per_step"]], dtype=torch.float64, device=dev)
                dist.all_reduce(fb, op=dist.ReduceOp.MAX)
                extras[name]["value"] = ns * world / (float(fb.item()) * 1e-3)
                extras[name]["ms_per_step_max_over_ranks"] = float(fb.item())
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu and not args.no_extras:
        r = cpu_leg(args.cpu_seconds, 1 << 21)
        cpu = {"value": r["value"], "unit": UNIT, "cores": r["cores"], "kind": "port", "cpu_model": cpu_model(),
               "sample": f"reference hh_step loop (oracle port of dynamics.py:443-529, fp32 mode) "
                         f"on {r['cores']} processes x {r['n_local']} neurons of the config-2 "
                         f"population for ~{args.cpu_seconds:.0f} s"}
    if world > 1:
        dist.barrier()
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
                "config": config_dict(args), "roofline": roof, "cpu_baseline": cpu,
                "e2e": extras.get("e2e"), "fwd_bwd": extras.get("fwd_bwd"),
                "fwd_bwd_bf16": extras.get("fwd_bwd_bf16"), "c5_network_100m": extras.get("c5_network_100m"),
                "cpu_model": cpu_model(),
                "c4_train_step": extras.get("c4_train_step"), "c5_network": extras.get("c5_network"),
                "morphology": extras.get("morphology"), "c5_replicas": extras.get("c5_replicas"),
"c1": extras.get("c1"),
                "gpu_launches": launches, "clocks": clk,
                "stimulus_ms_share": stim_ms / sum(step_ms)}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
