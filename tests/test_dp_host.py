"""Data-parallel gradient averaging of configs 3/4 over a
world-2 gloo group on CPU: layer.allreduce_gradients must leave every rank
with the mean of the ranks' gradients, in one flat bucket."""

import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2601_21407_b200.layer import allreduce_gradients


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = torch.Generator().manual_seed(100 + rank)
    params = [torch.nn.Parameter(torch.zeros(s)) for s in ((7, 5), (5,), (3, 2, 4))]
    for p in params:
        p.grad = torch.randn(p.shape, generator=g)
    frozen = torch.nn.Parameter(torch.zeros(3))     # no gradient: skipped
    flat = allreduce_gradients(params + [frozen])
    assert flat is not None and flat.numel() == sum(p.numel() for p in params)
    np.save(out % rank, np.concatenate([p.grad.reshape(-1).numpy() for p in params]))
    dist.destroy_process_group()


def test_allreduce_gradients_world2_averages(tmp_path):
    out = str(tmp_path / "g%d.npy")
    port = 29600 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    g0, g1 = np.load(out % 0), np.load(out % 1)
    ref = []
    for r in range(2):
        g = torch.Generator().manual_seed(100 + r)
        ref.append(np.concatenate([torch.randn(s, generator=g).reshape(-1).numpy()
                                   for s in ((7, 5), (5,), (3, 2, 4))]))
    mean = (ref[0] + ref[1]) / 2
    assert np.array_equal(g0, g1)
    assert np.allclose(g0, mean, rtol=1e-6, atol=1e-7)


def test_allreduce_gradients_single_process_is_noop():
    p = torch.nn.Parameter(torch.zeros(3))
    p.grad = torch.ones(3)
    assert allreduce_gradients([p]) is None and torch.equal(p.grad, torch.ones(3))
