"""Worker of tests/test_ep_gpu.py::test_peer_memory_ep_across_two_processes (2 ranks spawned on
ONE GPU, gloo for the host side): the peer-memory expert-parallel data path with REAL CUDA IPC
peer tables -- rows stored into the other process's receive block, GEMM2 reductions into the
other process's residual stream -- and the device barriers replaced by host barriers (kernels
of two processes on one GPU must never wait on each other). Each rank checks its token shard
against the single-device forward of the whole batch, bit for bit."""
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist


def main(rank: int, world: int, port: int, out: str) -> None:
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from paper_2605_11537_b200 import _lib
    from paper_2605_11537_b200._dev import ptr, stream_ptr
    from paper_2605_11537_b200.ep import CudaEpKernels
    from paper_2605_11537_b200.router_oracle import ToyMoeParams, _device_moe, _run_layers_device

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    L, E, d, F, T = 2, 16, 256, 512, 600
    rng = np.random.default_rng(42)
    params = ToyMoeParams(rng.normal(size=(L, E, d)).astype(np.float32),
                          (rng.normal(size=(L, E, F, d)) / np.sqrt(d)).astype(np.float32),
                          (rng.normal(size=(L, E, d, F)) / np.sqrt(F)).astype(np.float32))
    pop = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    e0 = rng.choice(E, size=world * T, p=pop / pop.sum())
    x0 = (params.router_weights[0][e0] * 0.05 + rng.normal(size=(world * T, d)) * 0.5).astype(np.float32)
    x_ref = torch.from_numpy(x0).to(dev)
    _run_layers_device(x_ref, _device_moe(params, dev))
    dm = _device_moe(params, dev)
    for lay in dm.layers:
        u2, v2 = lay.U.clone(), lay.V.clone()
        _lib.call("mp_tile_kmajor", ptr(u2), ptr(lay.U), E, F, d, _lib.size_query("mp_ffn_up_bn", F), stream_ptr())
        _lib.call("mp_tile_kmajor", ptr(v2), ptr(lay.V), E, d, F, _lib.size_query("mp_ffn_down_bn", d), stream_ptr())
        lay.tiled = 1
    res = torch.from_numpy((rng.integers(0, 3, size=(L, E))).astype(np.int32)).to(dev)
    k = CudaEpKernels(dm.layers, T, world, rank, world * (int(res.sum(1).max()) + E) + E, peer_cap=T, p2p=True)
    k.connect(None)
    x = torch.from_numpy(x0[rank * T:(rank + 1) * T].copy()).to(dev)

    def host_barrier():
        torch.cuda.synchronize()
        dist.barrier()

    for l in range(L):
        route = k.route(x, l)
        counts = k.counts(route)
        k.allgather_counts_peer(counts, barrier=False)  # peer stores into every rank's C_all
        host_barrier()
        parts = [torch.empty_like(counts.cpu()) for _ in range(world)]
        dist.all_gather(parts, counts.cpu())
        ok_counts = bool(torch.equal(k.C_all.cpu(), torch.stack(parts)))
        if not ok_counts:
            raise SystemExit("peer all-gather of the counts differs from gloo's")
        plan = k.plan(route, k.C_all, res[l])
        k.register_stream(x)
        k.dispatch_peer(x, plan)
        host_barrier()
        k.expert_ffn_peer(plan, l)
        host_barrier()
    ok = int(k.overflow.item()) == 0 and bool(torch.equal(x, x_ref[rank * T:(rank + 1) * T]))
    # the strided form (rows of n words into row-major (rows, G * n) buffers): the engine's
    # all-gather of the predicted assignments
    a = torch.randint(0, 1 << 20, (3, 50), dtype=torch.int32, device=dev, generator=torch.Generator(dev).manual_seed(rank))
    g_a = torch.zeros(3, world * 50, dtype=torch.int32, device=dev)
    t_a = k._mem.table(g_a)
    host_barrier()
    _lib.call("mp_peer_allgather_i32", ptr(a), 3, 50, rank, world, ptr(t_a), world * 50, stream_ptr())
    host_barrier()
    parts = [torch.empty(3, 50, dtype=torch.int32) for _ in range(world)]
    dist.all_gather(parts, a.cpu())
    ok = ok and bool(torch.equal(g_a.cpu(), torch.cat(parts, 1)))
    dist.barrier()
    with open(f"{out}.{rank}", "w") as f:
        f.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
