"""Grouped-FFN probe: GEMM1/GEMM2 time vs routing structure (T=16384, E=128, d=768, F=3072)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


def main():
    dev = require_device()
    T, E, d, F = 16384, 128, 768, 3072
    U = (torch.randn(E * F, d, device=dev) / 30).bfloat16()
    V = (torch.randn(E * d, F, device=dev) / 55).bfloat16()
    Ut, Vt = torch.empty_like(U), torch.empty_like(V)
    _lib.call("mp_tile_kmajor", ptr(U), ptr(Ut), E, F, d, 256, stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(V), ptr(Vt), E, d, F, _lib.size_query("mp_ffn_down_bn", d), stream_ptr())
    x = torch.randn(T, d, device=dev)
    rng = np.random.default_rng(0)
    w = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    cases = {
        "balanced": (np.repeat(np.arange(E), T // E), None, 1),
        "zipf_split": (rng.choice(E, size=T, p=w / w.sum()), None, 1),
        "zipf_off": (rng.choice(E, size=T, p=w / w.sum()), None, 0),
    }
    fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
    ws = torch.empty(fb, dtype=torch.uint8, device=dev)
    for name, (route, _, split) in cases.items():
        r = torch.from_numpy(route.astype(np.int32)).to(dev)
        se = torch.arange(E, dtype=torch.int32, device=dev)
        i32 = dict(dtype=torch.int32, device=dev)
        tor = torch.empty(T, **i32)
        pn = E + T // 128 + 1
        prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
        nb = _lib.size_query("mp_segments_workspace_bytes", T, E)
        sws = torch.empty(nb, dtype=torch.uint8, device=dev)
        for tiled, (u, v) in ((1, (Ut, Vt)), (3, (Ut, Vt)), (5, (Ut, Vt))):
            if tiled == 5 and not split:
                continue
            pn = 2 * (E + T // 128 + 1)
            prow, prows = torch.empty(pn, **i32), torch.empty(pn, **i32)
            _lib.call("mp_segments_from_slots", ptr(r), ptr(se), T, E, E, split | (tiled & 2), ptr(tor), ptr(prow),
                      ptr(prows), ptr(eb), ptr(sws), nb, stream_ptr())
            _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())
            t1 = timeit(lambda: _lib.call("mp_ffn_up", T, d, F, E, ptr(u), tiled, ptr(prow), ptr(prows), ptr(eb),
                                          ptr(ws), fb, stream_ptr()), iters=10)
            y = x.clone()
            t2 = timeit(lambda: _lib.call("mp_ffn_down", ptr(y), T, d, F, E, ptr(v), tiled, ptr(tor), ptr(prow),
                                          ptr(prows), ptr(eb), ptr(ws), fb, stream_ptr()), iters=10)
            npieces = int(eb[-1].item())
            b1 = E * F * d * 2 + T * d * 2 + T * F * 2
            b2 = E * F * d * 2 + T * F * 2 + T * d * 8
            print(f"{name:11s} tiled={tiled} pieces={npieces:4d}  up {t1:6.1f}us ({b1 / t1 / 1e3:5.0f} GB/s)  "
                  f"down {t2:6.1f}us ({b2 / t2 / 1e3:5.0f} GB/s)")


if __name__ == "__main__":
    main()
