"""Time one SRU layer (projection GEMM + scan passes) at the bench shape (T=16384, d=768)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


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

    def run():
        _lib.call("mp_sru_layer", ptr(xb), ptr(x), ptr(w), ptr(b), T, d, None, ptr(h32), ptr(h16), None, ptr(nf),
                  ptr(ws), n, stream_ptr())

    print(f"sru layer: {timeit(run, iters=20):.1f} us")

    def scan():
        _lib.call("mp_sru_scan", ptr(x), T, d, None, ptr(h32), ptr(h16), None, ptr(nf), ptr(ws), n, stream_ptr())

    print(f"sru scan: {timeit(scan, iters=20):.1f} us")
    import os
    out = os.environ.get("SRU_PROBE_OUT")
    if out:  # for cross-mode comparisons
        torch.save(h32.cpu(), out)


if __name__ == "__main__":
    main()
