"""GPU tests of the config-5 network (ring input, HH step, fixed-point
delivery): raster parity with the reference's run_network, and bit-exact
invariance under sharding the population over P ranks (emulated on one GPU:
every rank's local step, then the concatenated bitmap to every rank)."""

import numpy as np
import pytest
import torch

from conftest import golden, requires_jit
from paper_2601_21407_b200 import network as N

pytestmark = pytest.mark.gpu


def _small():
    g = golden("cortex_small")
    return g, N.build_network(float(g["scale"]), int(g["seed"]))


def test_fp64_network_reproduces_reference_raster(cuda):
    g, topo = _small()
    cfg = N.REST_CONFIG
    hb = N.HostBackground(topo, N.make_background(cfg), cfg.dt, np.random.default_rng(int(g["run_seed"])))
    net = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float64, background="host", host_bg=hb)
    steps = int(round(float(g["duration_ms"]) / cfg.dt))
    t, i = net.run(steps)
    order = np.lexsort((i, t))
    ref = np.lexsort((g["spike_id"], g["spike_t"]))
    assert np.array_equal(i[order], g["spike_id"][ref])
    assert np.allclose(t[order], g["spike_t"][ref])


def _run_sharded(topo, cfg, world, steps, dtype, cuda):
    nets = [N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, rank=r, world=world, background="philox",
                            seed=5) for r in range(world)]
    per = N.words_per_rank(topo.n_neurons, world)
    total = (topo.n_neurons + 31) // 32
    rows = []
    for _ in range(steps):
        allw = torch.cat([net.advance_local()[:per] for net in nets])[:total].contiguous()
        for net in nets:
            net.deliver(allw)
        rows.append(allw.clone())
    return torch.stack(rows).cpu().numpy(), [net.v.cpu().numpy() for net in nets]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_sharding_is_bit_exact(cuda, dtype):
    _, topo = _small()
    cfg = N.REST_CONFIG
    ref, v1 = _run_sharded(topo, cfg, 1, 300, dtype, cuda)
    assert ref.any()
    for world in (2, 4, 7):
        got, vs = _run_sharded(topo, cfg, world, 300, dtype, cuda)
        assert np.array_equal(got, ref), world
        assert np.array_equal(np.concatenate(vs), v1[0])


def test_philox_background_moments(cuda):
    """The device compound-Poisson drive has the reference's moments:
    mean lam*mu, variance lam*(mu^2 + sigma^2) per neuron-step (cortex.py:225-232)."""
    _, topo = _small()
    cfg = N.REST_CONFIG
    net = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float64, background="philox", seed=9)
    net.decay = 0.0                       # psp = this step's background only
    samples = []
    for _ in range(400):
        net._input()
        samples.append(net.cur[:net.n].clone())
        net.t += 1
    x = torch.stack(samples).cpu().numpy()
    lam = N.background_lambda(topo, N.make_background(cfg), cfg.dt)
    mu, sd = cfg.bg_mean, cfg.bg_std
    for k, p in enumerate(topo.populations):
        xs = x[:, p.offset:p.offset + p.size]
        L = lam[p.offset]
        assert abs(xs.mean() - L * mu) < 0.02 * L * mu
        assert abs(xs.var() - L * (mu * mu + sd * sd)) < 0.05 * L * (mu * mu + sd * sd)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_graph_replay_equals_eager_steps(cuda, dtype):
    """CortexNetwork.advance (CUDA graph of S steps, step index on the device)
    must reproduce step() bit for bit: rasters, membrane state and ring."""
    _, topo = _small()
    cfg = N.REST_CONFIG
    a = N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, background="philox", seed=3)
    b = N.CortexNetwork(topo, cfg, device=cuda, dtype=dtype, background="philox", seed=3)
    steps = 250                       # 3 graph replays of 64 + 58 eager device steps
    rows = torch.stack([a.step().clone() for _ in range(steps)])
    rec = torch.empty((steps, b.words_global), dtype=torch.int32, device=cuda)
    b.advance(steps, steps_per_graph=64, record=rec)
    assert rows.any()
    assert torch.equal(rows, rec)
    assert torch.equal(a.v, b.v) and torch.equal(a.g, b.g) and torch.equal(a.ring, b.ring)
    assert a.t == b.t == steps
    # and continuing after a replay (t on the device resynchronised)
    more = torch.stack([a.step().clone() for _ in range(70)])
    rec2 = torch.empty((70, b.words_global), dtype=torch.int32, device=cuda)
    b.advance(70, steps_per_graph=64, record=rec2)
    assert torch.equal(more, rec2)


def test_run_network_reproduces_reference_spike_records(cuda, tmp_path):
    """run_network (host background: the reference's RNG stream) reproduces the
    reference rasters, rest-state and with a thalamic transient, and the
    SpikeRecord statistics / ndjson output (cortex.py:319-464)."""
    g, topo = _small()
    rec = N.run_network(topo, N.REST_CONFIG, float(g["duration_ms"]), seed=int(g["run_seed"]))
    o, r = np.lexsort((rec.neuron_ids, rec.times_ms)), np.lexsort((g["spike_id"], g["spike_t"]))
    assert np.array_equal(rec.neuron_ids[o], g["spike_id"][r]) and np.allclose(rec.times_ms[o], g["spike_t"][r])
    h = golden("cortex_thalamic")
    topo_t = N.build_network(0.02, 0, N.THALAMIC_CONFIG)
    thal = {"t_on_ms": 4.0, "duration_ms": 10.0, "rate_hz": 120.0, "weight": 0.22, "weight_std": 0.022}
    rec = N.run_network(topo_t, N.THALAMIC_CONFIG, 20.0, seed=3, warmup_ms=2.0, thalamic=thal)
    assert np.array_equal(rec.neuron_ids, h["spike_id"]) and np.allclose(rec.times_ms, h["spike_t"], rtol=0, atol=1e-12)
    for pop in ("L4e", "L2/3e", "L6i"):
        key = pop.replace("/", "")
        assert rec.pop_rate(pop) == float(h[f"rate_{key}"])
        assert np.array_equal(rec.rate_quartiles(pop), h[f"quart_{key}"])
        cv = rec.isi_cv(pop)
        assert (np.isnan(cv) and np.isnan(h[f"cv_{key}"])) or cv == float(h[f"cv_{key}"])
        assert np.array_equal(rec.rate_histogram(pop, 2.0)[1], h[f"hist_{key}"])
    fn = tmp_path / "r.ndjson"
    rec.to_ndjson(fn)
    assert fn.read_text() == str(h["ndjson"])


def test_run_network_philox_graph_path(cuda):
    """The device-background path (graph replay) runs and fires; same record type."""
    _, topo = _small()
    rec = N.run_network(topo, N.REST_CONFIG, 30.0, seed=2, background="philox", dtype=np.float32)
    assert isinstance(rec, N.SpikeRecord) and rec.times_ms.size > 0
    assert rec.times_ms.max() <= 30.0 + 1e-9


def test_delay_impulse_and_dale_signs(cuda):
    """SPEC known answers of step_network: one forced presynaptic spike with
    delay d gives a postsynaptic current first nonzero exactly d steps later;
    excitatory rows deliver >= 0, inhibitory <= 0 (Dale)."""
    _, topo = _small()
    pops = topo.populations
    for k, p in enumerate(pops):
        w = topo.syn_weight[topo.syn_offsets[p.offset]:topo.syn_offsets[p.offset + p.size]]
        assert (w >= 0).all() if p.name.endswith("e") else (w <= 0).all()
    cfg = N.REST_CONFIG
    net = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float64, background="philox", seed=0)
    src = int(np.argmax(np.diff(topo.syn_offsets)))          # the source with most synapses
    lo, hi = topo.syn_offsets[src], topo.syn_offsets[src + 1]
    tgt, dly = topo.syn_target[lo:hi], topo.syn_delay[lo:hi]
    d_min = int(dly.min())
    words = torch.zeros(net.words_global, dtype=torch.int32, device=cuda)
    words[src // 32] = int(np.int32(np.uint32(1 << (src % 32))))
    net.deliver(words)                                       # spike of `src` at step 0
    ring = net.ring.cpu().numpy()
    for d in range(net.depth):
        row = ring[(d) % net.depth]
        hit = np.flatnonzero(row)
        exp_t = np.unique(tgt[dly == d])
        assert np.array_equal(hit, exp_t), d
    assert ring[d_min % net.depth].any() and not ring[0].any()


def test_zero_drive_stays_at_rest_and_rest_rates_match_reference(cuda):
    """No background and no activity: no spikes (rates 0).  The rest
    configuration at scale 0.1 with the device (Philox) background reproduces
    the reference's per-population rates from its own RNG stream (golden: the
    reference rest_state_run, 1 s after 200 ms warm-up) within 10%: the same
    compound-Poisson process, a different random stream."""
    from dataclasses import replace
    ka = golden("known_answers")
    topo = N.build_network(0.1, 0)
    quiet = replace(N.REST_CONFIG, bg_rate_hz=0.0)
    rec = N.run_network(topo, quiet, 50.0, seed=1, background="philox", dtype=np.float32)
    assert rec.times_ms.size == 0
    rec = N.run_network(topo, N.REST_CONFIG, 1200.0, seed=1, warmup_ms=200.0, background="philox",
                        dtype=np.float32)
    rates = np.array([rec.pop_rate(p.name) for p in topo.populations])
    ref = ka["rest_rates"]
    assert np.all(np.abs(rates - ref) <= 0.1 * ref + 0.2), (rates, ref)


def test_replicas_reproduce_single_network_runs(cuda):
    """CortexReplicas: replica r (seed + r) is bit-identical to a lone
    CortexNetwork run with seed + r (SPEC data-parallel batching)."""
    _, topo = _small()
    cfg = N.REST_CONFIG
    R, steps = 5, 200
    rep = N.CortexReplicas(topo, cfg, R, device=cuda, dtype=np.float32, seed=7)
    rec = torch.empty((steps, R, rep.words), dtype=torch.int32, device=cuda)
    rep.advance(steps, steps_per_graph=32, record=rec)
    assert rec.any()
    for r in (0, 3, 4):
        single = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float32, background="philox", seed=7 + r)
        rows = torch.stack([single.step().clone() for _ in range(steps)])
        assert torch.equal(rows, rec[:, r, :rows.shape[1]]), r
        assert torch.equal(single.v, rep.v[r * rep.n_pad:r * rep.n_pad + topo.n_neurons])


@requires_jit
@pytest.mark.parametrize("cap,nopair", [(None, False), ("3", False), (None, True)])
def test_persistent_kernel_equals_graph_path(cuda, monkeypatch, cap, nopair):
    """advance() on one rank with float32 neurons runs the persistent
    cooperative kernel (hhb_cortex_run); it must equal the graph path bit for
    bit -- rasters, state, PSP and ring -- also when a step's spikes need
    several delivery rounds (HHB_NET_CAP=3)."""
    _, topo = _small()
    cfg = N.REST_CONFIG
    if cap:
        monkeypatch.setenv("HHB_NET_CAP", cap)
    if nopair:   # the ring path of odd populations (no 16-byte pairs)
        monkeypatch.setenv("HHB_NET_NOPAIR", "1")
    a = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float32, background="philox", seed=11)
    b = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float32, background="philox", seed=11)
    assert a.persistent_ok()
    steps = 300
    ra = torch.empty((steps, a.words_global), dtype=torch.int32, device=cuda)
    a.advance(steps, record=ra)
    assert not getattr(a, "_no_persist", False), "the persistent path fell back"
    monkeypatch.setenv("HHB_NET_GRAPH", "1")
    assert not b.persistent_ok()
    rb = torch.empty_like(ra)
    b.advance(steps, steps_per_graph=64, record=rb)
    assert ra.any() and int(ra.ne(0).sum()) > 50
    assert torch.equal(ra, rb)
    for x, y in ((a.v, b.v), (a.g, b.g), (a.psp, b.psp), (a.ring, b.ring)):
        assert torch.equal(x, y)
    # continuing: unrecorded (ping-pong) persistent run, then eager steps
    monkeypatch.delenv("HHB_NET_GRAPH")
    a.advance(37)
    rows = torch.stack([b.step().clone() for _ in range(37)])
    assert torch.equal(a.words[:a.words_global], rows[-1]) and torch.equal(a.v, b.v)
    assert a.t == b.t == steps + 37


def test_spike_events_match_numpy_unpack(cuda):
    """hhb_spike_event_counts / hhb_spike_events == NumPy nonzero over the
    unpacked raster (order included), with a partial last word and empty rows."""
    rng = np.random.default_rng(4)
    T, n = 57, 1000
    W = (n + 31) // 32
    raw = (rng.random((T, W * 32)) < 0.03)
    raw[5] = False
    raw[:, n:] = True                      # bits past n must be ignored
    bits = np.packbits(raw, axis=1, bitorder="little").view(np.int32)
    st, nid = N.spike_events(torch.from_numpy(bits.copy()).to(cuda), n)
    t_ref, n_ref = np.nonzero(raw[:, :n])
    assert np.array_equal(st, t_ref) and np.array_equal(nid, n_ref)
    e_t, e_n = N.spike_events(torch.zeros((3, W), dtype=torch.int32, device=cuda), n)
    assert e_t.size == 0 and e_n.size == 0


def test_step_level_api_reproduces_reference_raster(cuda):
    """init_network_state / step_network / background_sample driven exactly as
    the reference's run_network loop (cortex.py:379-438) reproduce its raster."""
    g, topo = _small()
    cfg = N.REST_CONFIG
    rng = np.random.default_rng(int(g["run_seed"]))
    params = cfg.resolved_neuron()
    bg = N.make_background(cfg)
    net = N.init_network_state(topo, cfg, device=cuda)
    steps = int(round(float(g["duration_ms"]) / cfg.dt))
    times, ids = [], []
    for t in range(steps):
        spikes = N.step_network(net, topo, bg, cfg, rng, params)
        nz = np.flatnonzero(spikes)
        times.append(np.full(nz.size, (t + 1) * cfg.dt))
        ids.append(nz)
    t_all, i_all = np.concatenate(times), np.concatenate(ids)
    assert np.array_equal(i_all, g["spike_id"]) and np.allclose(t_all, g["spike_t"])
    assert net.t == steps and net.neuron.v.shape == (topo.n_neurons,) and net.psp.shape == (topo.n_neurons,)


def test_spike_buffer_matches_reference_semantics(cuda):
    """SpikeBuffer.enqueue / drain (cortex.py:238-256) in fixed point."""
    buf = N.SpikeBuffer(5, 7, device=cuda)
    buf.enqueue(3, np.array([1, 1, 6]), np.array([0.5, 0.25, -1.0]), np.array([1, 1, 4]))
    assert np.allclose(buf.ring[4], [0, 0.75, 0, 0, 0, 0, 0]) and np.allclose(buf.ring[2, 6], -1.0)
    assert np.allclose(buf.drain(4), [0, 0.75, 0, 0, 0, 0, 0]) and not buf.ring[4].any()
    assert np.allclose(buf.drain(7)[6], -1.0)
    with pytest.raises(Exception):
        N.SpikeBuffer(0, 3, device=cuda)


@pytest.mark.parametrize("graph", [False, True])
def test_non_finite_state_is_reported_with_its_step(cuda, monkeypatch, graph):
    """A non-finite membrane potential in the device network sets first_bad to
    the step that produced it (persistent kernel and graph path alike), which
    run_network turns into NumericalOverflowError (dynamics.py:526-527)."""
    from paper_2601_21407_b200.errors import NumericalOverflowError
    _, topo = _small()
    if graph:
        monkeypatch.setenv("HHB_NET_GRAPH", "1")
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float32, background="philox", seed=2)
    net.advance(10)
    assert int(net.first_bad.item()) == 2 ** 63 - 1
    net.psp[17] = float("inf")
    net.advance(5)
    assert int(net.first_bad.item()) == 10
    with pytest.raises(NumericalOverflowError):
        N._raise_if_bad(net.first_bad)


@requires_jit
def test_persistent_replicas_equal_graph_replicas(cuda, monkeypatch):
    """CortexReplicas in persistent launches (groups of <= 16 replicas) equal
    the graph path bit for bit, across a group boundary (R = 19)."""
    _, topo = _small()
    cfg = N.REST_CONFIG
    R, steps = 19, 120
    monkeypatch.setenv("HHB_NET_REPLICAS_PERSIST", "1")
    a = N.CortexReplicas(topo, cfg, R, device=cuda, dtype=np.float32, seed=4)
    b = N.CortexReplicas(topo, cfg, R, device=cuda, dtype=np.float32, seed=4)
    assert a.persistent_ok()
    ra = torch.empty((steps, R, a.words), dtype=torch.int32, device=cuda)
    a.advance(steps, record=ra)
    assert not getattr(a, "_no_persist", False), "the persistent path fell back"
    monkeypatch.setenv("HHB_NET_GRAPH", "1")
    rb = torch.empty_like(ra)
    b.advance(steps, steps_per_graph=40, record=rb)
    assert ra.any() and torch.equal(ra, rb)
    for x, y in ((a.v, b.v), (a.g, b.g), (a.psp, b.psp), (a.ring, b.ring)):
        assert torch.equal(x, y)


def test_record_buffer_shape_is_checked(cuda):
    """The persistent path writes n_steps * words int32 at a row pitch of
    exactly `words`: a record of the wrong row width, too few rows or another
    rank is refused (UsageError), a taller one is accepted."""
    from paper_2601_21407_b200.errors import UsageError
    _, topo = _small()
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float32, background="philox", seed=2)
    W = net.words_global
    for shape in ((10, W + 3), (9, W), (10, 1)):
        with pytest.raises(UsageError):
            net.advance(10, record=torch.zeros(shape, dtype=torch.int32, device=cuda))
    with pytest.raises(UsageError):
        net.advance(10, record=torch.zeros((10, W), dtype=torch.int64, device=cuda))
    tall = torch.zeros((15, W), dtype=torch.int32, device=cuda)
    net.advance(10, record=tall)
    assert not tall[10:].any()


@requires_jit
def test_graphs_captured_before_segment_sort_are_dropped(cuda, monkeypatch):
    """A graph captured on the unsorted synapse arrays must not be replayed
    after the persistent path re-sorted them (the old buffers are freed)."""
    _, topo = _small()
    monkeypatch.setenv("HHB_NET_GRAPH", "1")
    a = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float32, background="philox", seed=3)
    b = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float32, background="philox", seed=3)
    a.advance(40, steps_per_graph=20)
    b.advance(40, steps_per_graph=20)
    monkeypatch.setenv("HHB_NET_GRAPH", "0")
    a.advance(30)                                   # persistent: sorts the rows
    assert not a._graphs
    monkeypatch.setenv("HHB_NET_GRAPH", "1")
    a.advance(40, steps_per_graph=20)               # recaptured on the sorted arrays
    b.advance(70, steps_per_graph=10)
    assert torch.equal(a.v, b.v) and torch.equal(a.ring, b.ring)


def test_persistent_replicas_report_non_finite_state(cuda, monkeypatch):
    from paper_2601_21407_b200.errors import NumericalOverflowError
    _, topo = _small()
    monkeypatch.setenv("HHB_NET_REPLICAS_PERSIST", "1")
    r = N.CortexReplicas(topo, N.REST_CONFIG, 2, device=cuda, dtype=np.float32, seed=4)
    r.advance(5)
    r.psp[3] = float("inf")
    with pytest.raises(NumericalOverflowError):
        r.advance(5)


def test_spec_acceptance8_compound_poisson_1e6_draws(cuda):
    """SPEC.md:576 acceptance 8 / :407: 10^6 draws of the device compound-Poisson
    sampler (hhb_cortex_input bg_mode 2, Philox keyed by (seed, neuron, step))
    at lam = 3, mu = 0.17, sigma = 0.017: sample mean within 1 % of lam mu and
    variance within 1 % of lam (mu^2 + sigma^2)."""
    from paper_2601_21407_b200 import _native as nat
    lib = nat.load()
    n, depth = 250_000, 2
    lam = torch.full((n,), 3.0, dtype=torch.float64, device=cuda)
    ring = torch.zeros((depth, n), dtype=torch.int64, device=cuda)
    psp = torch.zeros(n, dtype=torch.float64, device=cuda)
    cur = torch.empty(n, dtype=torch.float64, device=cuda)
    draws = []
    for t in range(4):                       # 4 steps x 250,000 neurons = 10^6 draws
        psp.zero_()
        nat.check(lib.hhb_cortex_input(1, n, t, depth, ring.data_ptr(), psp.data_ptr(), 0.0, 2, None,
                                       lam.data_ptr(), 0.17, 0.017, 2024, 0, None, cur.data_ptr(), 1.0,
                                       torch.cuda.current_stream().cuda_stream), "cortex_input")
        draws.append(cur.clone())
    x = torch.cat(draws).cpu().numpy()
    assert x.size == 10 ** 6
    mean, var = 3 * 0.17, 3 * (0.17 ** 2 + 0.017 ** 2)
    assert abs(x.mean() - mean) < 0.01 * mean, x.mean()
    assert abs(x.var() - var) < 0.01 * var, x.var()
    # the trivial cases of SPEC.md:405-406: lam = 0 gives 0; sigma = 0 gives N mu
    lam.zero_()
    psp.zero_()
    nat.check(lib.hhb_cortex_input(1, n, 9, depth, ring.data_ptr(), psp.data_ptr(), 0.0, 2, None, lam.data_ptr(),
                                   0.17, 0.017, 2024, 0, None, cur.data_ptr(), 1.0,
                                   torch.cuda.current_stream().cuda_stream), "cortex_input")
    assert torch.count_nonzero(cur).item() == 0
    lam.fill_(3.0)
    psp.zero_()
    nat.check(lib.hhb_cortex_input(1, n, 9, depth, ring.data_ptr(), psp.data_ptr(), 0.0, 2, None, lam.data_ptr(),
                                   0.17, 0.0, 2024, 0, None, cur.data_ptr(), 1.0,
                                   torch.cuda.current_stream().cuda_stream), "cortex_input")
    k = (cur / 0.17).cpu().numpy()
    assert np.allclose(k, np.round(k), atol=1e-9)


# ---------------------------------------------------------------- thalamic drive on the device

def _philox4x32(c, key):
    """Philox-4x32-10 on uint64-held uint32 arrays (Salmon et al. 2011), the
    generator of hh_kernels.cuh / jit.cu, restated for the test."""
    M = 0xFFFFFFFF
    c0, c1, c2, c3 = (np.asarray(x, np.uint64) & M for x in c)
    k0, k1 = np.uint64(key[0] & M), np.uint64(key[1] & M)
    for _ in range(10):
        p0 = np.uint64(0xD2511F53) * c0
        p1 = np.uint64(0xCD9E8D57) * c2
        c0, c1, c2, c3 = ((p1 >> np.uint64(32)) ^ c1 ^ k0) & M, p1 & M, ((p0 >> np.uint64(32)) ^ c3 ^ k1) & M, p0 & M
        k0 = (k0 + np.uint64(0x9E3779B9)) & M
        k1 = (k1 + np.uint64(0xBB67AE85)) & M
    return c0, c1, c2, c3


def _thalamic_table(topo, seed=3):
    cfg = N.THALAMIC_CONFIG
    thal = {"t_on_ms": 2.0, "duration_ms": 10.0, "rate_hz": 400.0, "weight": cfg.bg_mean, "weight_std": cfg.bg_std}
    return N._thalamic_setup(topo, thal, 20.0, cfg.dt, np.random.default_rng(seed))


def test_device_thalamic_drive_matches_restated_philox(cuda):
    """hhb_thalamic_drive (float64) equals, bit for bit, the sum in row order
    of the weights of the synapses whose Philox word (seed ^ salt, synapse / 4,
    step) is below lam 2^32 -- the device form of cortex.py:423-428 -- and is
    0 outside [t_on, t_off)."""
    _, topo = _small()
    targets, weights, lam, lo, hi = _thalamic_table(topo)
    assert targets.size > 100
    net = N.CortexNetwork(topo, N.THALAMIC_CONFIG, device=cuda, dtype=np.float64, background="philox", seed=9)
    net.set_thalamic(targets, weights, lam, lo, hi)
    order = np.argsort(targets, kind="stable")
    tg, wg = targets[order], weights[order]
    thr = min(2 ** 32 - 1, int(np.floor(lam * 2.0 ** 32)))
    key = (net.seed ^ net.THAL_SALT) & (2 ** 64 - 1)
    ids = np.arange(tg.size, dtype=np.uint64)
    for t in (lo - 1, lo, lo + 3, hi - 1, hi):
        net.t = t
        got = net._thalamic().cpu().numpy()
        want = np.zeros(topo.n_neurons)
        if lo <= t < hi:
            g = ids >> np.uint64(2)
            words = _philox4x32((g, g >> np.uint64(32), np.full_like(g, t), np.zeros_like(g)),
                                (key & 0xFFFFFFFF, key >> 32))
            wd = np.choose((ids & np.uint64(3)).astype(np.int64), words)
            fire = wd < thr
            for k in np.flatnonzero(fire):           # row order = sorted-target order
                want[tg[k]] += wg[k]
            assert fire.any()
        assert np.array_equal(got, want), t


@requires_jit
def test_thalamic_persistent_graph_eager_and_shards_agree(cuda, monkeypatch):
    """With the device thalamic drive, the persistent kernel, the CUDA-graph
    path and eager steps give the same rasters and state bit for bit, and so
    does a 2-rank sharding (the draws are keyed by global synapse id)."""
    _, topo = _small()
    targets, weights, lam, lo, hi = _thalamic_table(topo)
    cfg = N.THALAMIC_CONFIG
    steps = 200

    def make(rank=0, world=1):
        net = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float32, background="philox", seed=13, rank=rank,
                              world=world)
        net.set_thalamic(targets, weights, lam, lo, hi)
        return net

    a = make()
    assert a.persistent_ok()
    ra = torch.empty((steps, a.words_global), dtype=torch.int32, device=cuda)
    a.advance(steps, record=ra)
    assert not getattr(a, "_no_persist", False)
    monkeypatch.setenv("HHB_NET_GRAPH", "1")
    b = make()
    rb = torch.empty_like(ra)
    b.advance(steps, record=rb)
    monkeypatch.delenv("HHB_NET_GRAPH")
    c = make()
    rc = torch.stack([c.step().clone() for _ in range(steps)])
    assert torch.equal(ra, rb) and torch.equal(ra, rc)
    for x, y, z in ((a.v, b.v, c.v), (a.psp, b.psp, c.psp)):
        assert torch.equal(x, y) and torch.equal(x, z)
    # the drive changes the run (against no thalamic input)
    d = N.CortexNetwork(topo, cfg, device=cuda, dtype=np.float32, background="philox", seed=13)
    rd = torch.empty_like(ra)
    d.advance(steps, record=rd)
    assert not torch.equal(ra, rd)
    # 2 ranks emulated on one GPU, sequentially (no kernel waits on another)
    nets = [make(r, 2) for r in range(2)]
    per = N.words_per_rank(topo.n_neurons, 2)
    total = (topo.n_neurons + 31) // 32
    rows = []
    for _ in range(steps):
        allw = torch.cat([net.advance_local()[:per] for net in nets])[:total].contiguous()
        for net in nets:
            net.deliver(allw)
        rows.append(allw.clone())
    assert torch.equal(torch.stack(rows), ra)


def test_thalamic_run_on_device_drives_l4(cuda):
    """run_network(thalamic=..., background="philox") runs through the device
    path (no host RNG loop): against the same run without thalamic input
    (identical background stream), a strong thalamic drive raises the L4
    spike count inside its window and leaves the run before it untouched;
    thalamic_stimulus_run(background="philox") runs end to end."""
    cfg = N.THALAMIC_CONFIG
    topo = N.build_network(0.05, 7, cfg)
    thal = {"t_on_ms": 60.0, "duration_ms": 20.0, "rate_hz": 3000.0, "weight": 2.0, "weight_std": 0.2}
    on = N.run_network(topo, cfg, 100.0, 8, thalamic=thal, background="philox", dtype=np.float32)
    off = N.run_network(topo, cfg, 100.0, 8, background="philox", dtype=np.float32)
    l4 = topo.pop_slice("L4e")

    def count(rec, a, b):
        t, ids = rec.times_ms, rec.neuron_ids
        return int(np.sum((ids >= l4.start) & (ids < l4.stop) & (t >= a) & (t < b)))

    pre_on, pre_off = on.times_ms < 60.0, off.times_ms < 60.0
    assert np.array_equal(on.times_ms[pre_on], off.times_ms[pre_off])
    assert np.array_equal(on.neuron_ids[pre_on], off.neuron_ids[pre_off])
    assert count(on, 60.0, 80.0) > 1.5 * count(off, 60.0, 80.0)
    rec = N.thalamic_stimulus_run(120.0, 0.05, 7, t_on_ms=60.0, warmup_ms=0.0, background="philox",
                                  dtype=np.float32)
    assert rec.times_ms.size > 0


def test_checked_kernels_run_clean(cuda):
    """HHB_JIT_CHECK=1 builds the generated kernels with device-side bounds and
    invariant checks that trap (compute-sanitizer is not available on this GPU
    pool): the persistent network kernel (grid barrier, delivery lists, tile
    segments, ring rows; with 3-spike delivery rounds and the thalamic drive)
    and the BPTT kernel (operand-ring slots) run through tools/sanitize_small.py
    without tripping any of them."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for env in ({"HHB_JIT_CHECK": "1"}, {"HHB_JIT_CHECK": "1", "HHB_NET_CAP": "3"}):
        for which in ("net", "bwd", "fwd"):
            out = subprocess.run([sys.executable, "tools/sanitize_small.py", which], cwd=root, capture_output=True,
                                 text=True, timeout=600, env={**os.environ, **env})
            assert out.returncode == 0 and "ok " + which in out.stdout, (env, which, out.stdout[-2000:],
                                                                      out.stderr[-2000:])
