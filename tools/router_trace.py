"""Per-CTA phase timeline of the fused router (diagnostic build -DMP_DIAG): when each x
k-block is issued, lands and has its operand in TMEM, and when the accumulator is complete,
averaged over the CTAs of one routing call at the bench shape (x resident in L2 or not).

usage: python tools/router_trace.py
"""
import ctypes
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200.build import PKG, build  # noqa: E402

lib = _lib.load_library(build(extra=["-DMP_DIAG"], out=PKG / "libmoempmc_trace.so"))
lib.mp_debug_router_trace.restype = ctypes.c_int
lib.mp_debug_router_trace.argtypes = [ctypes.c_void_p]

from paper_2605_11537_b200._dev import ptr, stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402


def main():
    cfg = PipelineConfig(num_layers=1)
    pipe = MoEPipeline(cfg)
    x = pipe.wl.batch(cfg.tokens)[0]
    lay = pipe.layers[0]
    T, d, E = cfg.tokens, cfg.d_model, cfg.num_experts
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    buf = np.zeros((160, 80), np.uint64)

    def call():
        _lib.call("mp_route_top1_hist", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                  ptr(pipe.route[0]), ptr(pipe.ws_exec), ptr(pipe.ws_router), pipe.ws_router_n, stream_ptr())

    for flushed in (False, True):
        for _ in range(5):
            if flushed:
                flush.zero_()
            call()
        torch.cuda.synchronize()
        _lib.check(lib.mp_debug_router_trace(buf.ctypes.data), "mp_debug_router_trace")
        n = (T + 127) // 128
        t = buf[:n].astype(np.int64)
        base = t[:, 0].min()
        rel = (t - base) / 1e3
        nkb = d // 64
        print(f"x {'flushed from L2' if flushed else 'in L2'}: {n} CTAs, span {rel[:, 75].max():.2f} us "
              f"(start spread {rel[:, 0].max():.2f}, setup done {np.median(rel[:, 1]):.2f})")
        print("   kb   issued   landed     read  tmem-free  stored  operand   (median over CTAs, us from the "
              "first CTA start; read/free/stored: converter warp 4)")
        for kb in range(min(nkb, 12)):
            print("   %2d " % kb + " ".join(f"{np.median(rel[:, c + kb]):8.2f}" for c in (2, 14, 26, 38, 50, 62)))
        print(f"   accumulator full {np.median(rel[:, 74]):.2f}, CTA end {np.median(rel[:, 75]):.2f} "
              f"(max {rel[:, 75].max():.2f})")


if __name__ == "__main__":
    with torch.cuda.stream(torch.cuda.Stream()):
        main()
