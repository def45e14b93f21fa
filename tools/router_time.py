"""Time the engine's routing call (mp_route_top1_hist) alone at the bench shape, x in L2 or not."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def main():
    cfg = PipelineConfig(num_layers=1)
    pipe = MoEPipeline(cfg)
    x = pipe.wl.batch(cfg.tokens)[0]
    lay = pipe.layers[0]
    T, d, E = cfg.tokens, cfg.d_model, cfg.num_experts
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def call():
        _lib.call("mp_route_top1_hist", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                  ptr(pipe.route[0]), ptr(pipe.ws_exec), ptr(pipe.ws_router), pipe.ws_router_n, stream_ptr())

    for _ in range(5):
        call()
    torch.cuda.synchronize()
    for flushed in (False, True):
        ts = []
        for _ in range(30):
            if flushed:
                flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            call()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        print(f"router {'(L2 flushed)' if flushed else '(x in L2)   '}: median {ts[15]:.1f} us  min {ts[0]:.1f} us")


if __name__ == "__main__":
    with torch.cuda.stream(torch.cuda.Stream()):
        main()
