"""CPU tests of the config-5 network host logic: the topology builder is pinned
to the reference's network (sha256 of its CSR arrays), the oracle network step
reproduces the reference's spike raster, and the sharded exchange protocol
(32-aligned shards, target-local synapse rows, bitmap all-gather over gloo,
world_size 2) gives exactly the single-rank result."""

import hashlib
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden
from oracle import hh_oracle as O
from paper_2601_21407_b200 import network as N


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def _small():
    g = golden("cortex_small")
    return g, N.build_network(float(g["scale"]), int(g["seed"]))


def test_topology_matches_reference():
    g, topo = _small()
    assert topo.n_neurons == int(g["n_neurons"]) and topo.n_synapses == int(g["n_synapses"])
    assert topo.max_delay == int(g["max_delay"])
    assert [p.size for p in topo.populations] == list(g["sizes"])
    for key, arr in (("offsets", topo.syn_offsets), ("target", topo.syn_target),
                     ("weight", topo.syn_weight), ("delay", topo.syn_delay)):
        assert _sha(arr) == str(g["sha_" + key]), key
    assert np.array_equal(topo.syn_target[:200], g["head_target"])
    assert np.array_equal(topo.syn_offsets, g["offsets"])


@pytest.mark.parametrize("n,world", [(1544, 2), (38586, 8), (100, 3), (31, 4), (64, 2)])
def test_shards_are_word_aligned_and_cover(n, world):
    prev = 0
    for r in range(world):
        lo, hi = N.shard_range(n, r, world)
        assert lo == prev and (lo % 32 == 0 or lo == n) and lo <= hi   # trailing shards may be empty
        prev = hi
    assert prev == n


def test_local_synapse_rows_partition_the_network():
    _, topo = _small()
    got = []
    for r in range(3):
        lo, hi = N.shard_range(topo.n_neurons, r, 3)
        off, tgt, w, d = N.local_synapses(topo, lo, hi)
        src = np.repeat(np.arange(topo.n_neurons), np.diff(off))
        got.append(np.stack([src, tgt.astype(np.int64) + lo, d], 1))
    got = np.concatenate(got)
    ref = np.stack([np.repeat(np.arange(topo.n_neurons), np.diff(topo.syn_offsets)),
                    topo.syn_target.astype(np.int64), topo.syn_delay], 1)
    key = lambda a: a[np.lexsort(a.T[::-1])]
    assert np.array_equal(key(got), key(ref))


def _oracle_run(topo, cfg, steps, seed, lo=0, hi=None, gather=None):
    """Oracle network (cortex.py:273-310) on neurons [lo, hi); `gather` maps the
    local spike vector to the global one (identity when unsharded)."""
    hi = topo.n_neurons if hi is None else hi
    p = cfg.resolved_neuron()
    rng = np.random.default_rng(seed)
    hb = N.HostBackground(topo, N.make_background(cfg), cfg.dt, rng)
    v, gt = O.rest_state(p, hi - lo)
    psp = np.zeros(hi - lo)
    ring = O.Ring(topo.max_delay + 1, hi - lo)
    off, tgt, w, d = N.local_synapses(topo, lo, hi)
    decay = np.exp(-cfg.dt / cfg.psp_tau_ms)
    times, ids = [], []
    for t in range(steps):
        bg = hb.sample()[lo:hi]
        psp = psp * decay + ring.pop(t)
        psp = psp + bg
        v, gt, sp = O.step(p, v, gt, psp, step_index=t)
        full = sp if gather is None else gather(sp)
        for s in np.flatnonzero(full):
            a, b = off[s], off[s + 1]
            if b > a:
                ring.push(t, tgt[a:b], w[a:b], d[a:b])
        nz = np.flatnonzero(full)
        times.append(np.full(nz.size, (t + 1) * cfg.dt))
        ids.append(nz)
    return np.concatenate(times), np.concatenate(ids)


def test_oracle_network_reproduces_reference_raster():
    g, topo = _small()
    steps = int(round(float(g["duration_ms"]) / N.REST_CONFIG.dt))
    t, i = _oracle_run(topo, N.REST_CONFIG, steps, int(g["run_seed"]))
    assert np.array_equal(i, g["spike_id"]) and np.allclose(t, g["spike_t"])
    assert i.size > 100


def _gloo_worker(rank, world, port, steps, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g, topo = _small()
    n = topo.n_neurons
    lo, hi = N.shard_range(n, rank, world)
    per = N.words_per_rank(n, world)

    def gather(local_spikes):
        words = np.zeros(per * 32, dtype=bool)
        words[:hi - lo] = local_spikes
        packed = torch.from_numpy(np.packbits(words, bitorder="little").view(np.int32).copy())
        allw = torch.empty(per * world, dtype=torch.int32)
        dist.all_gather_into_tensor(allw, packed)
        bits = np.unpackbits(allw.numpy().view(np.uint8), bitorder="little").astype(bool)
        return bits[:n]

    t, i = _oracle_run(topo, N.REST_CONFIG, steps, int(g["run_seed"]), lo, hi, gather)
    if rank == 0:
        np.save(out, np.stack([t, i]))
    dist.destroy_process_group()


def test_sharded_exchange_gloo_world2_equals_single_rank(tmp_path):
    g, topo = _small()
    steps = 200
    out = str(tmp_path / "r.npy")
    port = 29500 + os.getpid() % 1000
    mp.spawn(_gloo_worker, args=(2, port, steps, out), nprocs=2, join=True)
    t2, i2 = np.load(out)
    t1, i1 = _oracle_run(topo, N.REST_CONFIG, steps, int(g["run_seed"]))
    assert np.array_equal(i2.astype(np.int64), i1) and np.allclose(t2, t1)
    assert i1.size > 100   # recurrent activity crosses the shard boundary


def test_background_sample_matches_reference_draws():
    """network.background_sample reproduces the reference's RNG call sequence."""
    from conftest import golden
    ka = golden("known_answers")
    out = N.background_sample(ka["bg_lam"], 0.11, 0.02, 40, np.random.default_rng(21))
    assert np.array_equal(out, ka["bg_sample"])
