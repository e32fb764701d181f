"""Multi-rank config-5 paths of the product:

* two processes in a gloo group, each running the product CortexNetwork for
  its shard with network.allgather_exchange (host-staged for gloo, so both may
  share the box's one GPU and no kernel waits on another process), reproduce
  the one-rank rasters and state bit for bit (cortex.py:273-310);
* the library exchange (hhb_spk_step: ncclAllGather + delivery in one C-ABI
  call) captured into advance()'s CUDA graphs, on a one-rank NCCL
  communicator, equals the single-rank path bit for bit, and its status /
  wait / abort plumbing works;
* bench.py's N > 1 branch runs end to end under torchrun with the gloo
  backend (2 ranks on one GPU)."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from conftest import golden
from paper_2601_21407_b200 import network as N

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _topo():
    g = golden("cortex_small")
    return N.build_network(float(g["scale"]), int(g["seed"]))


def test_two_rank_product_exchange_matches_one_rank(cuda, tmp_path):
    steps, world = 200, 2
    port = _free_port()
    outs = [str(tmp_path / f"r{r}.npz") for r in range(world)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "exchange_worker.py"), str(r), str(world),
                               str(port), outs[r], str(steps)], cwd=ROOT, stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(world)]
    logs = [p.communicate(timeout=600)[0] for p in procs]
    assert all(p.returncode == 0 for p in procs), logs
    topo = _topo()
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float64, background="philox", seed=3)
    ref = torch.stack([net.step().clone() for _ in range(steps)]).cpu().numpy()
    v1 = net.v.cpu().numpy()
    assert ref.any()
    res = [np.load(o) for o in outs]
    for r in res:
        assert np.array_equal(r["words"], ref)
    assert np.array_equal(np.concatenate([r["v"] for r in res]), v1)


def test_library_exchange_in_cuda_graphs_equals_single_rank(cuda):
    from paper_2601_21407_b200 import _native as nat
    if not nat.load().hhb_spk_exchange_available():
        pytest.fail("libnccl.so.2 not loadable on the GPU box")
    topo = _topo()
    steps = 256
    W = (topo.n_neurons + 31) // 32
    ref_net = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float32, background="philox", seed=4)
    ref = torch.zeros((steps, W), dtype=torch.int32, device=cuda)
    ref_net.advance(steps, record=ref)
    ex = N.LibraryExchange(topo.n_neurons, rank=0, world=1)
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=cuda, dtype=np.float32, background="philox", seed=4,
                          exchange=ex)
    assert not net.persistent_ok()                # the graph path with hhb_spk_step captured
    got = torch.zeros((steps, W), dtype=torch.int32, device=cuda)
    net.advance(steps, record=got)
    assert ref.any() and torch.equal(got, ref)
    assert torch.equal(net.v, ref_net.v) and torch.equal(net.ring, ref_net.ring)
    ex.check()
    ex.wait()
    ex.abort()
    from paper_2601_21407_b200.errors import ExchangeError
    with pytest.raises(ExchangeError):
        ex(net.words, net.gwords)


def test_bench_multi_rank_branch_runs_under_torchrun_gloo(cuda):
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--backend", "gloo", "--steps", "1",
           "--warmup", "3", "--neurons", "262144", "--sim-steps", "200", "--chunk", "100", "--no-cpu",
           "--legs", "fwd_bwd,c4_train_step,c5_network"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0
    for k in ("fwd_bwd", "c4_train_step", "c5_network"):
        assert "error" not in line[k], line[k]
        assert line[k]["value"] > 0
    assert "gloo" in line["c5_network"]["path"]
    assert "ms_per_step_max_over_ranks" in line["c4_train_step"]
