"""One rank of the multi-process spike-exchange test -- TEST INFRASTRUCTURE
(run by tests/test_gpu_exchange.py as a subprocess).

    python tests/exchange_worker.py RANK WORLD PORT OUT.npz STEPS

Joins a gloo group on 127.0.0.1:PORT, builds the product CortexNetwork for its
neuron shard of the small golden network (float64, device Philox background)
with the product all-gather (network.allgather_exchange; gloo stages the
bitmap through host memory, so the ranks may share one GPU without any kernel
waiting on another rank's), steps it STEPS times through CortexNetwork.step,
and saves the global spike words of every step and its shard's final V.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
import torch.distributed as dist

from paper_2601_21407_b200 import network as N


def main():
    rank, world, port, out, steps = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], int(sys.argv[5])
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    g = np.load(os.path.join(ROOT, "tests", "golden", "cortex_small.npz"))
    topo = N.build_network(float(g["scale"]), int(g["seed"]))
    dev = torch.device("cuda", 0)
    net = N.CortexNetwork(topo, N.REST_CONFIG, device=dev, dtype=np.float64, rank=rank, world=world,
                          exchange=N.allgather_exchange(topo.n_neurons), background="philox", seed=3)
    rows = [net.step().clone() for _ in range(steps)]
    np.savez(out, words=torch.stack(rows).cpu().numpy(), v=net.v.cpu().numpy(), lo=net.lo, hi=net.hi)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
