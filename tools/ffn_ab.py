"""A/B the grouped expert GEMM pair inside the real step graph (BASELINE config 3).

For every variant (a set of environment variables read by the C-ABI at capture time) the
step is re-captured twice: once plain (timed step, CUDA events around K replays) and once
with event nodes around every layer's GEMM1 / GEMM2 (per-launch durations). Variants are
interleaved over several rounds so box drift hits all of them alike.

usage: python tools/ffn_ab.py [--rounds 3] [--steps 20] VAR=VAL[+VAR=VAL] ...   ("-" = no env)
"""
import argparse
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import DeviceEvent, MoEPipeline, PipelineConfig  # noqa: E402


def parse(v):
    if v == "-":
        return {}
    return dict(kv.split("=", 1) for kv in v.split("+"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=3)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--replication", default="on")
    ap.add_argument("--predictor", default="constructed")
    ap.add_argument("variants", nargs="+")
    args = ap.parse_args()
    cfg = PipelineConfig(replication=args.replication, predictor=args.predictor)
    pipe = MoEPipeline(cfg)
    L = cfg.num_layers
    batches = [pipe.wl.batch(cfg.tokens)[0] for _ in range(4)]
    x = torch.empty_like(batches[0])
    _lib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, 1.0, stream_ptr())
    for k in range(3):
        x.copy_(batches[k % 4])
        pipe.step(x)
    torch.cuda.synchronize()
    ref_out = None
    res = {v: {"step": [], "g1": [], "g2": []} for v in args.variants}
    for rnd in range(args.rounds):
        for v in args.variants:
            env = parse(v)
            old = {k: os.environ.get(k) for k in env}
            os.environ.update(env)
            try:
                ev = [[DeviceEvent() for _ in range(3)] for _ in range(L)]
                g = pipe.capture(x)
                gev = pipe.capture(x, ev)
            finally:
                for k, o in old.items():
                    if o is None:
                        os.environ.pop(k, None)
                    else:
                        os.environ[k] = o
            for k in range(3):
                x.copy_(batches[k % 4])
                g.replay()
            # output of one fixed batch: every variant must agree bitwise
            x.copy_(batches[0])
            g.replay()
            torch.cuda.synchronize()
            out = x.clone()
            if ref_out is None:
                ref_out = out
            same = bool(torch.equal(out, ref_out))
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            for k in range(args.steps):
                x.copy_(batches[k % 4])
                g.replay()
            e.record()
            torch.cuda.synchronize()
            res[v]["step"].append(s.elapsed_time(e) / args.steps)
            g1, g2 = [], []
            for k in range(3):
                x.copy_(batches[k % 4])
                gev.replay()
                torch.cuda.synchronize()
                g1 += [ev[l][0].elapsed_ms(ev[l][1]) * 1e3 for l in range(L)]
                g2 += [ev[l][1].elapsed_ms(ev[l][2]) * 1e3 for l in range(L)]
            res[v]["g1"].append(statistics.mean(g1))
            res[v]["g2"].append(statistics.mean(g2))
            print(f"round {rnd} {v:40s} step {res[v]['step'][-1]:.3f} ms  gemm1 {res[v]['g1'][-1]:6.1f} us  "
                  f"gemm2 {res[v]['g2'][-1]:6.1f} us  bitwise_same={same}", flush=True)
            del g, gev
    print("summary (median over rounds)")
    for v in args.variants:
        r = res[v]
        print(f"  {v:40s} step {statistics.median(r['step']):.3f} ms  gemm1 {statistics.median(r['g1']):6.1f} us  "
              f"gemm2 {statistics.median(r['g2']):6.1f} us  pair {statistics.median(r['g1']) + statistics.median(r['g2']):6.1f} us")


if __name__ == "__main__":
    with torch.cuda.stream(torch.cuda.Stream()):  # capturable (non-legacy) stream
        main()
