"""One steady-state engine step (eager launches) bracketed by cudaProfilerStart/Stop, for
`ncu --profile-from-start off` launch lists and full captures of chosen kernels."""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replication", default="on")
    ap.add_argument("--experts", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None)
    ap.add_argument("--capacity", type=int, default=None)
    args = ap.parse_args()
    kw = {k: v for k, v in (("num_experts", args.experts), ("num_layers", args.layers), ("capacity", args.capacity))
          if v is not None}
    cfg = PipelineConfig(replication=args.replication, **kw)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipe = MoEPipeline(cfg)
        batches = [pipe.wl.batch(cfg.tokens)[0] for _ in range(2)]
        x = torch.empty_like(batches[0])
        _lib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, 1.0, s.cuda_stream)
        for k in range(3):
            x.copy_(batches[k % 2])
            pipe.step(x)
        torch.cuda.synchronize()
        x.copy_(batches[1])
        torch.cuda.synchronize()
        torch.cuda.profiler.start()
        pipe.step(x)
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
    print("launches in the step:", pipe.launches_per_step)


if __name__ == "__main__":
    main()
