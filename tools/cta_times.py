"""Per-CTA start/end times of layer l's GEMM1 and GEMM2 (eager, after steady-state steps),
with each CTA's unit count and weight/activation bytes: load balance of the static
round-robin schedule.

usage: python tools/cta_times.py [--layer 0]
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def cta_times(n):
    t0 = np.zeros(n, np.uint64)
    t1 = np.zeros(n, np.uint64)
    _lib.call("mp_debug_cta_times", t0.ctypes.data, t1.ctypes.data, n)
    return t0.astype(np.int64), t1.astype(np.int64)


def report(name, t0, t1, units_of_cta, rows_of_cta):
    base = t0.min()
    s, e = (t0 - base) / 1e3, (t1 - base) / 1e3
    print(f"{name}: span {e.max():.1f} us  start max {s.max():.1f}  end min {e.min():.1f} "
          f"p10 {np.percentile(e, 10):.1f} p50 {np.percentile(e, 50):.1f} p90 {np.percentile(e, 90):.1f}")
    for k in sorted(set(units_of_cta)):
        m = units_of_cta == k
        print(f"   {m.sum():3d} CTAs with {k} units: end {e[m].min():.1f}..{e[m].max():.1f} us "
              f"(mean {e[m].mean():.1f}); rows mean {rows_of_cta[m].mean():.0f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", type=int, default=0)
    ap.add_argument("--replication", default="on")
    args = ap.parse_args()
    cfg = PipelineConfig(replication=args.replication)
    pipe = MoEPipeline(cfg)
    T, d, F, E = cfg.tokens, cfg.d_model, cfg.d_ff, cfg.num_experts
    batches = [pipe.wl.batch(T)[0] for _ in range(2)]
    x = torch.empty_like(batches[0])
    sp = stream_ptr()
    _lib.call("mp_l2_persist", x.data_ptr(), x.numel() * 4, 1.0, sp)
    for k in range(4):
        x.copy_(batches[k % 2])
        pipe.step(x)
    torch.cuda.synchronize()
    l = args.layer
    lay = pipe.layers[l]
    eb = pipe.exp_begin[l].cpu().numpy()
    prows = pipe.piece_rows[l].cpu().numpy()
    P = int(eb[-1])
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    print(f"layer {l}: {P} pieces, touched experts {(eb[1:] > eb[:-1]).sum()}, rows {prows[:P].sum()}")
    for name, nt, rev in (("GEMM1", F // 256, False), ("GEMM2", d // _lib.size_query("mp_ffn_down_bn", d), True)):
        # unit u -> piece (expert-major, slice, piece), CTA = u % grid
        units = []
        for e in range(E):
            b, c = eb[e], eb[e + 1] - eb[e]
            for s in range(nt):
                for p in range(c):
                    units.append(b + p)
        units = np.array(units)
        if rev:
            units = units[::-1]
        nu = len(units)
        cta = np.arange(nu) % nsm
        upc = np.bincount(cta, minlength=nsm)
        rpc = np.bincount(cta, weights=prows[units], minlength=nsm)
        for rep in range(3):
            if name == "GEMM1":
                _lib.call("mp_ffn_up", T, d, F, E, ptr(lay.U), lay.tiled, ptr(pipe.piece_row[l]),
                          ptr(pipe.piece_rows[l]), ptr(pipe.exp_begin[l]), ptr(pipe.ws_ffn), pipe.ws_ffn_n, sp)
            else:
                y = x.clone()
                _lib.call("mp_ffn_down", ptr(y), T, d, F, E, ptr(lay.V), lay.tiled, ptr(pipe.tok_of_row[l]),
                          ptr(pipe.piece_row[l]), ptr(pipe.piece_rows[l]), ptr(pipe.exp_begin[l]), ptr(pipe.ws_ffn),
                          pipe.ws_ffn_n, sp)
            torch.cuda.synchronize()
        t0, t1 = cta_times(nsm)
        print(f"{name}: {nu} units over {nsm} CTAs")
        report(name, t0, t1, upc, rpc)


if __name__ == "__main__":
    with torch.cuda.stream(torch.cuda.Stream()):
        main()
