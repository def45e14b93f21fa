"""Per-unit timeline of layer l's grouped expert GEMMs (diagnostic build with -DMP_DIAG).

Every unit of the static round-robin schedule is stamped by its CTA's producer (first load
issued) and MMA issuer (first k-block landed, last k-block issued). A unit's cost is the
time between the MMA finishing the previous unit of the same CTA and finishing this one.
Units are classed by their expert: "hot" (the expert has >= 2 replica pieces, so its weight
slices are shared through L2 by several units) or "cold" (a single piece: its weight slices
stream from HBM once). Reports the mean cost per class and, per 10 us window, how many units
of each class were running and what they cost -- whether cold units are slower when the
window is full of cold units (a shared HBM limit) or equally slow everywhere (a per-SM limit).

usage: python tools/unit_trace.py [--layer 0]
"""
import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200.build import PKG, build  # noqa: E402

TRACE_LIB = build(extra=["-DMP_DIAG"], out=PKG / "libmoempmc_trace.so")
lib = _lib.load_library(TRACE_LIB)
lib.mp_debug_unit_trace.restype = ctypes.c_int
lib.mp_debug_unit_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]

from paper_2605_11537_b200._dev import ptr, stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def unit_list(eb, E, nt, rev):
    units, hot = [], []
    for e in range(E):
        b, c = eb[e], eb[e + 1] - eb[e]
        for _ in range(nt):
            for p in range(c):
                units.append(b + p)
                hot.append(c >= 2)
    units, hot = np.array(units), np.array(hot)
    return (units[::-1], hot[::-1]) if rev else (units, hot)


def analyse(name, tr, units, hot, prows):
    nu = len(units)
    t0, t1, t2, cta = (tr[k][:nu].astype(np.int64) for k in range(4))
    base = t0.min()
    t0, t1, t2 = (t0 - base) / 1e3, (t1 - base) / 1e3, (t2 - base) / 1e3
    start = np.zeros(nu)
    for c in np.unique(cta):
        idx = np.where(cta == c)[0]
        idx = idx[np.argsort(t2[idx])]
        prev = np.concatenate([[t1[idx[0]]], t2[idx[:-1]]])
        start[idx] = prev
    cost = t2 - start
    print(f"{name}: {nu} units, span {t2.max():.1f} us; hot {hot.sum()} cold {(~hot).sum()}")
    for lab, m in (("hot", hot), ("cold", ~hot)):
        print(f"   {lab:4s}: cost mean {cost[m].mean():5.2f} us  p10 {np.percentile(cost[m], 10):5.2f}  "
              f"p50 {np.percentile(cost[m], 50):5.2f}  p90 {np.percentile(cost[m], 90):5.2f}  rows mean "
              f"{prows[units[m]].mean():5.1f}  (sum {cost[m].sum():7.0f} SM-us)")
    print("   window    hot-busy cold-busy  hot-cost cold-cost   (SM-us of each class running, mean unit cost)")
    w = 10.0
    for a in np.arange(0, t2.max(), w):
        b = a + w
        ov = np.clip(np.minimum(t2, b) - np.maximum(start, a), 0, None)
        in_w = (t2 >= a) & (t2 < b)
        hc = cost[in_w & hot].mean() if (in_w & hot).any() else float("nan")
        cc = cost[in_w & ~hot].mean() if (in_w & ~hot).any() else float("nan")
        print(f"   {a:5.0f}-{b:<5.0f} {ov[hot].sum():8.0f} {ov[~hot].sum():9.0f} {hc:9.2f} {cc:9.2f}")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layer", type=int, default=0)
    args = ap.parse_args()
    cfg = PipelineConfig()
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
    print(f"layer {l}: {int(eb[-1])} pieces, rows {prows[:int(eb[-1])].sum()}")
    buf = np.zeros((4, 8192), np.uint64)
    for name, nt, rev in (("GEMM1", F // 256, False), ("GEMM2", d // _lib.size_query("mp_ffn_down_bn", d), True)):
        units, hot = unit_list(eb, E, nt, rev)
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
        _lib.check(lib.mp_debug_unit_trace(buf.ctypes.data, 8192), "mp_debug_unit_trace")
        analyse(name, buf, units, hot, prows)


if __name__ == "__main__":
    with torch.cuda.stream(torch.cuda.Stream()):
        main()
