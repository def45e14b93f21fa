"""In-graph time of every C-ABI call of one engine step (events recorded between calls
inside the captured CUDA graph -- no profiler, real overlap/launch gaps included).

usage: python tools/step_profile.py [--replication on|off|split] [--steps N]
"""
import argparse
import collections
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200.engine import DeviceEvent, MoEPipeline, PipelineConfig  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--replication", default="on")
    ap.add_argument("--steps", type=int, default=10)
    args = ap.parse_args()
    cfg = PipelineConfig(replication=args.replication)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipe = MoEPipeline(cfg)
        emb, _, _ = pipe.wl.batch(cfg.tokens)
        x = emb.clone()
        pipe.step(x)  # configure kernels
        torch.cuda.synchronize()
        # as bench.py: keep the residual stream persisting in L2 (stream attribute, inherited by graph nodes)
        _lib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, 1.0, torch.cuda.current_stream().cuda_stream)
        marks = []  # (name, event) after each call
        orig = _lib.call
        capturing = {"on": False}

        def call(name, *a):
            rc = orig(name, *a)
            if capturing["on"] and not name.startswith(("mp_event", "mp_graph")) and "workspace" not in name:
                ev = DeviceEvent()
                ev.record(a[-1] if isinstance(a[-1], int) else torch.cuda.current_stream().cuda_stream)
                marks.append((name, ev))
            return rc

        _lib.call = call
        import paper_2605_11537_b200.engine as eng
        eng._lib.call = call
        first = DeviceEvent()
        sp = torch.cuda.current_stream().cuda_stream
        orig("mp_graph_begin", sp)
        capturing["on"] = True
        first.record(sp)
        pipe.step(x)
        capturing["on"] = False
        import ctypes
        ex = ctypes.c_void_p()
        orig("mp_graph_end", sp, ctypes.byref(ex))
        for _ in range(20):  # warm up (clocks, caches)
            x.copy_(emb)
            orig("mp_graph_launch", ex, sp)
        torch.cuda.synchronize()
        tot = collections.defaultdict(float)
        cnt = collections.Counter()
        for _ in range(args.steps):
            x.copy_(emb)  # fresh input each step (outside the timed events)
            orig("mp_graph_launch", ex, sp)
            torch.cuda.synchronize()
            prev = first
            for name, ev in marks:
                tot[name] += prev.elapsed_ms(ev) * 1e3
                cnt[name] += 1
                prev = ev
        step_us = sum(tot.values()) / args.steps
        print(f"step {step_us:.1f} us  ({len(marks)} calls)")
        for name, us in sorted(tot.items(), key=lambda kv: -kv[1]):
            n = cnt[name] // args.steps
            print(f"  {us / args.steps:8.1f} us/step  {n:3d} calls  {us / args.steps / n:7.1f} us/call  "
                  f"{100 * us / args.steps / step_us:5.1f}%  {name}")


if __name__ == "__main__":
    main()
