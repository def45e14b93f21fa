"""Where the expert-parallel step spends its time at world size 1: GPU busy time (sum of
kernel and memcpy durations from the CUDA profiler) vs the step's wall time, and the
top device operations. usage: python tools/ep_profile.py [--force-collectives]"""
import socket
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def main():
    force = "--force-collectives" in sys.argv
    if force:
        import torch.distributed as dist
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                                device_id=torch.device("cuda", 0))
    cfg = PipelineConfig()
    pipe = MoEPipeline(cfg)
    pipe.enable_expert_parallel()
    pipe.force_collectives = force
    emb = pipe.wl.batch(cfg.tokens)[0]
    x = emb.clone()
    for _ in range(3):
        x.copy_(emb)
        pipe.step(x)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    n = 5
    for _ in range(n):
        x.copy_(emb)
        pipe.step(x)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e3
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        x.copy_(emb)
        pipe.step(x)
        torch.cuda.synchronize()
    evs = [e for e in prof.events() if e.device_type.name == "CUDA"]
    busy = sum(e.device_time for e in evs) / 1e3
    print(f"EP step (world 1, collectives {'forced' if force else 'skipped'}): wall {wall:.2f} ms/step, "
          f"GPU busy {busy:.2f} ms ({busy / wall * 100:.0f} %)")
    print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=18))


if __name__ == "__main__":
    main()
