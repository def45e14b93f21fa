"""Per-block phase timeline of the single-pass SRU scan (diagnostic build -DMP_DIAG) at the
bench shape (T = 16384, d = 768): when each block (ticket order) has its chunk maps, its
carry-in (after the look-back) and its replay done -- medians and spreads over the blocks.

usage: python tools/scan_trace.py
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
lib.mp_debug_scan_trace.restype = ctypes.c_int
lib.mp_debug_scan_trace.argtypes = [ctypes.c_void_p]
lib.mp_debug_scan_trace_reset.restype = ctypes.c_int

from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402


def main():
    dev = require_device()
    T, d = 16384, 768
    x = torch.randn(T, d, device=dev) * 0.5
    xb = x.bfloat16()
    w = (torch.randn(3 * d, d, device=dev) / d ** 0.5).bfloat16()
    b = torch.randn(3 * d, device=dev) * 0.1
    h32 = torch.empty(T, d, device=dev)
    h16 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    nf = torch.zeros(1, dtype=torch.int32, device=dev)
    n = _lib.size_query("mp_sru_workspace_bytes", T, d)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    buf = np.zeros((1024, 4), np.uint64)
    for _ in range(3):
        _lib.call("mp_sru_project", ptr(xb), ptr(w), ptr(b), T, d, ptr(ws), n, stream_ptr())
        lib.mp_debug_scan_trace_reset()
        _lib.call("mp_sru_scan", ptr(x), T, d, None, ptr(h32), ptr(h16), None, ptr(nf), ptr(ws), n, stream_ptr())
        torch.cuda.synchronize()
    _lib.check(lib.mp_debug_scan_trace(buf.ctypes.data), "mp_debug_scan_trace")
    nb = int((buf[:, 0] > 0).sum())
    t = buf[:nb].astype(np.int64)
    rel = (t - t[:, 0].min()) / 1e3
    ph1, look, rep = rel[:, 1] - rel[:, 0], rel[:, 2] - rel[:, 1], rel[:, 3] - rel[:, 2]
    print(f"{nb} blocks, span {rel[:, 3].max():.2f} us (start spread {rel[:, 0].max():.2f})")
    for name, v in (("chunk maps", ph1), ("look-back", look), ("replay", rep)):
        print(f"  {name:10s} median {np.median(v):6.2f} us  p10 {np.percentile(v, 10):6.2f}  p90 "
              f"{np.percentile(v, 90):6.2f}  max {v.max():6.2f}")
    nstr = d // 128
    for q in (0, nb // 4, nb // 2, 3 * nb // 4, nb - 1):
        print(f"  ticket {q:4d} (block {q // nstr:3d} of its strip): start {rel[q, 0]:6.2f} maps {rel[q, 1]:6.2f} "
              f"carry {rel[q, 2]:6.2f} end {rel[q, 3]:6.2f}")


if __name__ == "__main__":
    with torch.cuda.stream(torch.cuda.Stream()):
        main()
