"""Where does the end-to-end (host buffers) throughput go? Times pinned H2D / D2H of one
batch alone and concurrently, and the captured step alone vs with copies in flight."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def timed(fn, stream, n=10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    a.record(stream)
    for _ in range(n):
        fn()
    b.record(stream)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def main():
    cfg = PipelineConfig()
    comp = torch.cuda.Stream()
    h2d, d2h = torch.cuda.Stream(), torch.cuda.Stream()
    with torch.cuda.stream(comp):
        pipe = MoEPipeline(cfg)
        emb, _, _ = pipe.wl.batch(cfg.tokens)
        x = emb.clone()
        _lib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, 1.0, comp.cuda_stream)
        pipe.step(x)
        g = pipe.capture(x)
        hin = emb.cpu().pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        dbuf = torch.empty_like(x)
        mb = hin.numel() * 4 / 1e6

        def h():
            with torch.cuda.stream(h2d):
                dbuf.copy_(hin, non_blocking=True)
        def dd():
            with torch.cuda.stream(d2h):
                hout.copy_(dbuf, non_blocking=True)
        t = timed(h, h2d)
        print(f"H2D {mb:.0f} MB: {t:.3f} ms ({mb / t:.1f} GB/s)")
        t = timed(dd, d2h)
        print(f"D2H {mb:.0f} MB: {t:.3f} ms ({mb / t:.1f} GB/s)")

        def both():
            h()
            dd()
        t = timed(both, d2h)
        print(f"H2D+D2H concurrent: {t:.3f} ms")

        def step():
            x.copy_(emb)
            g.replay()
        t = timed(step, comp)
        print(f"step alone (incl. 50 MB d2d reset): {t:.3f} ms")

        def step_with_copies():
            h()
            dd()
            x.copy_(emb)
            g.replay()
        t = timed(step_with_copies, comp)
        print(f"step with concurrent H2D+D2H: {t:.3f} ms")


if __name__ == "__main__":
    main()
