"""Worker process for the CPU (gloo) expert-parallel tests: runs ``ExpertParallelMoE``
with the numpy oracle kernels on its token shard and saves the results."""

import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def make_problem(seed, L=2, E=8, d=16, F=12, T=48):
    rng = np.random.default_rng(seed)
    router = rng.normal(size=(L, E, d)).astype(np.float32)
    eu = (rng.normal(size=(L, E, F, d)) / np.sqrt(d)).astype(np.float32)
    ev = (rng.normal(size=(L, E, d, F)) / np.sqrt(F)).astype(np.float32)
    # skew the routing: a few experts get most tokens
    router[:, 0] *= 2.5
    router[:, 1] *= 1.8
    x = rng.normal(size=(T, d)).astype(np.float32)
    res = rng.integers(0, 4, size=(L, E)).astype(np.int32)  # warm residency: replicas 0..3
    return router, eu, ev, x, res


def run_worker(rank, world, port, seed, outdir):
    from oracle.ep_oracle import OracleEpKernels
    from paper_2605_11537_b200.ep import ExpertParallelMoE

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    router, eu, ev, x, res = make_problem(seed)
    T = x.shape[0]
    lo, hi = rank * T // world, (rank + 1) * T // world
    xl = torch.from_numpy(x[lo:hi].copy())
    k = OracleEpKernels(router, eu, ev, rank, world)
    ep = ExpertParallelMoE(k, router.shape[0], router.shape[1])
    ep.res.copy_(torch.from_numpy(res))
    slots = []
    for l in range(router.shape[0]):
        ep.layer(l, xl)
        slots.append(k._p["slot_of_token"])
    np.savez(os.path.join(outdir, f"{rank}.npz"), x=xl.numpy(), res=ep.res.numpy(),
             slots=np.stack(slots))
    dist.barrier()
    dist.destroy_process_group()
