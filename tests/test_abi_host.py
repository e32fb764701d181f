"""CPU tests of the boundary: the C-ABI library loads and exports every symbol
include/hhb200.h declares, the ctypes structs match the C layout, and the
host-side logic (parameter validation, plans, stats) mirrors the reference.
No kernel is launched here."""

import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest
import torch

from conftest import ROOT, golden
from paper_2601_21407_b200 import _native as nat
from paper_2601_21407_b200 import adjoint as A
from paper_2601_21407_b200 import defaults as DF
from paper_2601_21407_b200 import dynamics as Dy
from paper_2601_21407_b200.errors import (ConfigurationError, NativeLibraryError,
                                          NumericalOverflowError, UsageError)

HEADER = os.path.join(ROOT, "include", "hhb200.h")


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hhb_[a-z0-9_]+)\s*\(", txt)))


def test_library_is_newer_than_its_sources():
    """A stale libhhb200.so would silently test old kernels."""
    lib_t = os.path.getmtime(nat.LIB_PATH)
    csrc = os.path.join(ROOT, "paper_2601_21407_b200", "csrc")
    srcs = [os.path.join(csrc, f) for f in os.listdir(csrc)] + [HEADER]
    stale = [s for s in srcs if os.path.getmtime(s) > lib_t]
    assert not stale, f"rebuild: python -m paper_2601_21407_b200._build ({stale})"


def test_library_exports_every_declared_symbol():
    lib = nat.load()
    names = _declared()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), f"{name} not exported"
        assert name in nat.SIGNATURES, f"{name} not typed in _native.SIGNATURES"
    assert lib.hhb_abi_version() == nat.ABI_VERSION


def test_symbol_visibility_with_nm():
    out = subprocess.run(["nm", "-D", "--defined-only", nat.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (hhb_[a-z0-9_]+)", out))
    assert set(_declared()) <= exported


def test_struct_layout_matches_c_header():
    src = r"""
    #include <stdio.h>
    #include <stddef.h>
    #include "hhb200.h"
    int main(void) {
      printf("%zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(hhb_rate_t), sizeof(hhb_gate_t),
             sizeof(hhb_channel_t), sizeof(hhb_params_t), sizeof(hhb_surrogate_t),
             offsetof(hhb_params_t, gates), offsetof(hhb_params_t, channels),
             offsetof(hhb_gate_t, exponent));
      return 0;
    }
    """
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "l.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "l")
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        vals = list(map(int, subprocess.run([exe], capture_output=True, text=True).stdout.split()))
    mine = [C.sizeof(nat.Rate), C.sizeof(nat.Gate), C.sizeof(nat.Channel), C.sizeof(nat.Params),
            C.sizeof(nat.Surrogate), nat.Params.gates.offset, nat.Params.channels.offset,
            nat.Gate.exponent.offset]
    assert vals == mine


def test_param_table_validation_matches_reference_errors():
    p = DF.na_kdr_cal_kca_params()
    P = nat.pack_hh(p)
    assert (P.n_gates, P.n_channels) == (6, 5)
    assert [P.gates[g].channel for g in range(6)] == [0, 0, 1, 3, 3, 4]
    assert (P.channels[2].gate_begin, P.channels[2].gate_count) == (3, 0)
    with pytest.raises(ConfigurationError):
        Dy.RateFn("tanh", 1.0, 0.0, 1.0)
    with pytest.raises(ConfigurationError):
        Dy.RateFn("exp", 1.0, 0.0, 0.0)
    with pytest.raises(ConfigurationError):
        Dy.GateSpec("g", Dy.RateFn("exp", 1, 0, 1), Dy.RateFn("exp", 1, 0, 1), -1)
    with pytest.raises(ConfigurationError):
        Dy.ChannelSpec("c", -1.0, 0.0)
    with pytest.raises(ConfigurationError):
        p.with_(c_m=0.0)
    with pytest.raises(ConfigurationError):
        p.with_(dt=-1.0)
    with pytest.raises(ConfigurationError):
        p.with_(channels=p.channels + (p.channels[0],))
    # C-side check (the same table, corrupted)
    P.channels[1].gate_begin = 5
    assert nat.load().hhb_check_params(C.byref(P)) == nat.EINVAL
    # more gates than the kernels carry in registers
    g = p.channels[0].gates[0]
    big = Dy.HHParams(1.0, (Dy.ChannelSpec("x", 1.0, 0.0, (g,) * 9),), -65.0, 0.0, 0.01)
    with pytest.raises(ConfigurationError):
        nat.pack_hh(big)


def test_dict_round_trip():
    p = DF.na_kdr_cal_kca_params(dt=0.02, rate_scale=1.5)
    q = Dy.HHParams.from_dict(p.to_dict())
    assert q == p.with_(dtype=np.float64)
    assert q.gate_layout == p.gate_layout and q.n_gates == 6
    with pytest.raises(ConfigurationError):
        Dy.HHParams.from_dict({"c_m": 1.0})


def test_plans_and_stats_match_reference_counts():
    ka = golden("known_answers")
    for (T, b), seg, cnt in zip(ka["plan_in"], ka["plan_seg"], ka["plan_count"]):
        pl = A.make_plan(int(T), int(b))
        assert pl.segment_length == seg and len(pl.stored_indices) == cnt
    with pytest.raises(UsageError):
        A.make_plan(0, 3)
    with pytest.raises(UsageError):
        A.CheckpointPlan(10, 2, (1, 3))
    with pytest.raises(UsageError):
        A.CheckpointPlan(10, 2, (0, 5))
    for case in ("bptt_rs", "bptt_squid_rect", "bptt_c2"):
        g = golden(case)
        T = g["i"].shape[0]
        seg = A.make_plan(T, int(g["budget"])).segment_length
        st = A._plan_stats(T, seg, False)
        assert (st.forward_calls, st.peak_stored_states) == (int(g["plan_calls"]), int(g["plan_peak"]))
        st = A._plan_stats(T, 1, True)
        assert (st.forward_calls, st.peak_stored_states) == (int(g["full_calls"]), int(g["full_peak"]))
    # T=400, budget 20 -> peak <= 40, forward calls <= 2T + budget
    st = A._plan_stats(400, A.make_plan(400, 20).segment_length, False)
    assert st.peak_stored_states <= 40 and st.forward_calls <= 2 * 400 + 20


def test_surrogate_spec_validation():
    assert A.default_surrogate(DF.squid_axon_params()).width == 16.25
    with pytest.raises(UsageError):
        A.SurrogateSpec("tanh", 1.0)
    with pytest.raises(UsageError):
        A.SurrogateSpec("rectangular", 0.0)


def test_errors_carry_step_index():
    e = NumericalOverflowError("membrane potential became non-finite", 12)
    assert e.step_index == 12 and "(step 12)" in str(e)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_product_path_fails_loudly_without_gpu():
    p = DF.squid_axon_params()
    with pytest.raises(NativeLibraryError):
        Dy.simulate(p, np.zeros((3, 2)), state0=Dy.NeuronState(np.full(2, -65.0), np.zeros((3, 2))))
    with pytest.raises(NativeLibraryError):
        Dy.gate_rates(p.channels[0].gates[0], np.zeros(3))


@pytest.mark.parametrize("mk", [lambda: DF.squid_axon_params(), lambda: DF.cortical_rs_params(rate_scale=1.4),
                                lambda: DF.na_kdr_cal_kca_params(),
                                lambda: Dy.HHParams(1.0, (Dy.ChannelSpec("leak", 0.1, -70.0),), -70.0, 0.0, 0.1)])
def test_jit_source_compiles_for_sm100a(mk, tmp_path):
    """The runtime-specialised float kernels (jit.cu) must compile for sm_100a
    for every channel structure; checked here with nvcc (no GPU needed)."""
    src = nat.jit_source(mk())
    assert "step_fwd" in src and "hh_bwd" in src and "hh_fwd_v4" in src
    f = tmp_path / "g.cu"
    f.write_text(src)
    r = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-cubin", "-O3", str(f),
                        "-o", str(tmp_path / "g.cubin")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]


def _mufu_ops(src: str, fn: str) -> int:
    # the merged forward is generated in paired (f32x2) form: ex2v / rcpv = one
    # MUFU op per neuron
    head = "F2 " + fn + "2(" if "F2 " + fn + "2(" in src else "float " + fn + "("
    body = src[src.index(head):]
    body = body[:body.index("\n}\n")]
    return sum(body.count(k) for k in ("ex2f_(", "rcpf_(", "ex2v<H>(", "rcpv<H>("))


@pytest.mark.parametrize("mk,tau,merged", [(lambda: DF.na_kdr_cal_kca_params(), 31, 20),
                                           (lambda: DF.cortical_rs_params(), 16, 10),
                                           (lambda: DF.squid_axon_params(), 15, 10)])
def test_merged_step_mufu_budget(mk, tau, merged):
    """jit.cu mg::plan_of: rates of equal |b| share one exp and each gate's
    divisions share one reciprocal (config 2: 8 shared exps + 6 decays + 6
    reciprocals = 20); the direct step keeps the reference's transcendental
    count."""
    src = nat.jit_source(mk())
    assert "// merged form off" not in src
    assert _mufu_ops(src, "step_fwd_m") == merged
    assert _mufu_ops(src, "step_fwd_s") == tau


def test_merged_step_window_and_fallback():
    """The merged form is used only inside the voltage window where every
    intermediate stays in float range; a table it cannot prove (a zero rate
    amplitude) keeps the direct step."""
    src = nat.jit_source(DF.na_kdr_cal_kca_params())
    line = next(l for l in src.splitlines() if "bool regular(" in l)
    assert "fabsf" in line
    m = Dy.RateFn("sigmoid", 0.0, -20.0, 5.0)
    ch = Dy.ChannelSpec("x", 1.0, -90.0, (Dy.GateSpec("c", m, Dy.RateFn("exp", 0.005, -65.0, 40.0), 1),))
    p = Dy.HHParams(1.0, (ch, Dy.ChannelSpec("leak", 0.1, -70.0)), -70.0, 0.0, 0.01)
    src = nat.jit_source(p)
    assert "// merged form off" in src and "step_fwd_m" not in src


def test_every_reference_public_name_exists():
    """Drop-in coverage: each public name of each reference module
    (tests/golden/api_names.json, written by oracle/make_golden.py from the
    reference package) exists in the same-named module here."""
    import importlib
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "api_names.json")
    api = json.load(open(path))
    missing = {m: [n for n in names if not hasattr(importlib.import_module("paper_2601_21407_b200." + m), n)]
               for m, names in api.items()}
    assert not any(missing.values()), missing
    assert sum(len(v) for v in api.values()) > 100


def test_new_entry_points_validate_arguments_without_a_gpu():
    """Argument checks of the late entry points return HHB_EINVAL before any
    CUDA call (so they run here, without a GPU), with a message."""
    lib = nat.load()
    P = Dy._table(DF.cortical_rs_params().with_(dtype=np.float32))
    E = nat.EINVAL
    # readout GEMV / gradient: negative sizes, NULL pointers, short workspace
    assert lib.hhb_readout_drive(nat.F64, -1, 2, 3, None, 0, 0, None, None, None, None) == E
    assert lib.hhb_readout_drive(nat.F64, 2, 2, 3, None, 6, 3, None, None, None, None) == E
    assert lib.hhb_readout_workspace(nat.F64, 64) == 296 * 65 * 8
    assert lib.hhb_readout_grad(nat.F64, 2, 2, 3, 1, 6, 3, 1, 1, 1, 1, 8, None) == E
    # spike events: more neurons than the bitmap holds
    assert lib.hhb_spike_event_counts(4, 2, 1, 65, 1, None) == E
    assert lib.hhb_spike_events(4, 2, 1, 64, None, 1, 1, None) == E
    # persistent network: replicas < 1, ld < n, bad bitmap width
    args = [C.byref(P), 0, 100, 100, 10, 0, 5, 1, 1, 0.9, 0, None, 0.0, 0.0, 0, 0, 1.0, 1, 1, 100, 1, 0, 4, 1,
            1, 1, 1, 1, 1, 1, None, None]
    assert lib.hhb_cortex_run_replicas(*args) == E
    args[1], args[2] = 1, 50
    assert lib.hhb_cortex_run_replicas(*args) == E
    args[2], args[22] = 100, 3
    assert lib.hhb_cortex_run_replicas(*args) == E
    assert b"cortex_run" in lib.hhb_last_error()
    # fused-MSE partials: a count for any population size
    assert lib.hhb_forward_partials(0) >= 1 and lib.hhb_forward_partials(10 ** 7) >= 10 ** 7 // 32


def test_integration_doc_maps_every_entry_point():
    """INTEGRATION.md names every symbol include/hhb200.h declares."""
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    missing = [n for n in _declared() if n not in doc]
    assert not missing, missing


@pytest.mark.parametrize("which", ["rs", "c2", "squid"])
def test_generated_modules_compile_for_sm100a_without_a_gpu(which):
    """Every NVRTC module the library generates (forward + backward, the
    persistent network kernel, its 4-replica form) compiles for sm_100a here,
    on the CPU (hhb_jit_cubin: NVRTC only, no device)."""
    import numpy as np
    from paper_2601_21407_b200 import defaults as DF
    p = {"rs": DF.cortical_rs_params(dt=0.1), "c2": DF.na_kdr_cal_kca_params(dt=0.01),
         "squid": DF.squid_axon_params(dt=0.01)}[which].with_(dtype=np.float32)
    for kind in ((0, 1, 2) if which == "rs" else (0,)):
        cubin = nat.jit_cubin(p, kind)
        assert cubin[:4] == b"\x7fELF" and len(cubin) > 10000


def test_forward_module_issues_paired_fp32_ops(tmp_path):
    """The merged forward step is generated in f32x2 form (jit.cu mg::pair):
    the 4-neurons/thread config-2 kernel issues FFMA2 / FMUL2 (two neurons per
    instruction) with at most a token spill (one slot, outside the step); the network module keeps the
    scalar step (FWD_PAIR 0)."""
    import shutil
    import subprocess
    import numpy as np
    from paper_2601_21407_b200 import defaults as DF
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    p = DF.na_kdr_cal_kca_params(dt=0.01).with_(dtype=np.float32)
    f = tmp_path / "fwd.cubin"
    f.write_bytes(nat.jit_cubin(p, -1 - (1 | 2 | 16)))        # FF_VO | FF_SO | FF_AL: the bench stream set
    sass = subprocess.run([tool, "-sass", "-fun", "hh_fwdp_v4", str(f)], capture_output=True, text=True).stdout
    assert sass.count("FFMA2 ") > 50 and sass.count("FMUL2 ") > 50
    assert sass.count("STL") + sass.count("LDL") <= 4
    src = nat.jit_source(p)
    assert "F2 step_fwd_m2(" in src and "#define FWD_PAIR 1" in src
