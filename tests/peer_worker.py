"""Worker of tests/test_ep_gpu.py::test_peer_memory_tables_map_another_process (spawned, 2 ranks
on ONE GPU, gloo for the host exchange): each rank fills a slice of its own buffer, maps the
other rank's slice through ep.PeerMemory (CUDA IPC) and copies it out with a plain gather
kernel. No kernel waits on another process."""
import sys

import torch
import torch.distributed as dist


def main(rank: int, world: int, port: int, out: str) -> None:
    sys.path.insert(0, str(__import__("pathlib").Path(__file__).resolve().parents[1]))
    from paper_2605_11537_b200 import _lib
    from paper_2605_11537_b200._dev import ptr, stream_ptr
    from paper_2605_11537_b200.ep import PeerMemory

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    n, d = 64, 256
    big = torch.zeros(n + 3, d, dtype=torch.bfloat16, device=dev)
    buf = big[3:]  # a view with a storage offset
    buf.copy_((torch.arange(n * d, device=dev).view(n, d) % 251 + 1000 * rank).to(torch.bfloat16))
    torch.cuda.synchronize()
    mem = PeerMemory(None, world, rank, dev)  # holds the mapped storages
    table = mem.table(buf)
    ok = int(table[rank].item()) == buf.data_ptr()
    other = 1 - rank
    got = torch.empty(n, d, dtype=torch.bfloat16, device=dev)
    idx = torch.arange(n, dtype=torch.int32, device=dev)
    _lib.call("mp_gather_rows_bf16", int(table[other].item()), n, d, ptr(idx), ptr(got), stream_ptr())
    torch.cuda.synchronize()
    want = (torch.arange(n * d, device=dev).view(n, d) % 251 + 1000 * other).to(torch.bfloat16)
    ok = ok and bool(torch.equal(got, want))
    dist.barrier()  # the owner keeps its buffer until the other rank has read it
    with open(f"{out}.{rank}", "w") as f:
        f.write("ok" if ok else "mismatch")
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4])
