"""A/B one grouped GEMM (up or down) between FFN kernel flags on a fixed routing -- for ncu captures.

usage: python tools/ffn_ab.py {up|down} {balanced|zipf} FLAGS [FLAGS ...]
"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


def main():
    which, case, flags = sys.argv[1], sys.argv[2], [int(f) for f in sys.argv[3:] if not f.startswith("--")]
    dev = require_device()
    import os
    T, E, d, F = int(os.environ.get("FFN_T", 16384)), 128, 768, 3072
    U = (torch.randn(E * F, d, device=dev) / 30).bfloat16()
    V = (torch.randn(E * d, F, device=dev) / 55).bfloat16()
    U0, V0 = U.clone(), V.clone()
    _lib.call("mp_tile_kmajor", ptr(U0), ptr(U), E, F, d, 256, stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(V0), ptr(V), E, d, F, _lib.size_query("mp_ffn_down_bn", d), stream_ptr())
    x = torch.randn(T, d, device=dev)
    rng = np.random.default_rng(0)
    w = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    route = np.repeat(np.arange(E), T // E) if case == "balanced" else rng.choice(E, size=T, p=w / w.sum())
    r = torch.from_numpy(route.astype(np.int32)).to(dev)
    se = torch.arange(E, dtype=torch.int32, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    tor = torch.empty(T, **i32)
    pn = 2 * (E + T // 128 + 1)
    prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
    nb = _lib.size_query("mp_segments_workspace_bytes", T, E)
    sws = torch.empty(nb, dtype=torch.uint8, device=dev)
    segs = {}
    for sm in (1, 3):  # split pieces; split + even piece count per expert (CTA-pair kernels)
        t_, pr_, pn_, eb_ = torch.empty(T, **i32), torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
        _lib.call("mp_segments_from_slots", ptr(r), ptr(se), T, E, E, sm, ptr(t_), ptr(pr_), ptr(pn_), ptr(eb_),
                  ptr(sws), nb, stream_ptr())
        segs[sm] = (t_, pr_, pn_, eb_)
    tor, prow, prows, eb = segs[1]
    fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
    ws = torch.empty(fb, dtype=torch.uint8, device=dev)
    _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())
    y = x.clone()
    for fl in flags:
        tor, prow, prows, eb = segs[3 if fl & 2 else 1]
        _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())

        def run():
            if which == "up":
                _lib.call("mp_ffn_up", T, d, F, E, ptr(U if fl & 1 else U0), fl, ptr(prow), ptr(prows), ptr(eb),
                          ptr(ws), fb, stream_ptr())
            else:
                _lib.call("mp_ffn_down", ptr(y), T, d, F, E, ptr(V if fl & 1 else V0), fl, ptr(tor), ptr(prow),
                          ptr(prows), ptr(eb), ptr(ws), fb, stream_ptr())
        print(f"{which} {case} flags={fl}: {timeit(run, iters=10):.1f} us", flush=True)
        torch.cuda.synchronize()
        cta_spread(f"  {which} {case}", units=(prows, eb, 12 if which == "up" else 3))
    torch.cuda.synchronize()



def cta_spread(label="", units=None):
    """Per-CTA start/end spread of the last grouped-GEMM launch (load-balance diagnostic)."""
    import ctypes

    n = 148
    t0 = (ctypes.c_ulonglong * n)()
    t1 = (ctypes.c_ulonglong * n)()
    _lib.call("mp_debug_cta_times", ctypes.cast(t0, ctypes.c_void_p).value, ctypes.cast(t1, ctypes.c_void_p).value, n)
    a, b = np.array(t0[:n], dtype=np.float64), np.array(t1[:n], dtype=np.float64)
    s = a.min()
    ends = np.sort(b - s) / 1e3
    print(f"{label} CTA end times (us from first start): min {ends[0]:.1f}  p10 {ends[14]:.1f}  median "
          f"{ends[74]:.1f}  p90 {ends[133]:.1f}  max {ends[-1]:.1f}; start spread {(a.max() - s) / 1e3:.1f}")
    if units is not None:  # static round-robin unit assignment (SegSched order) vs end time
        prows, eb, nt = units
        ebh = eb.cpu().numpy()
        pr = prows.cpu().numpy()
        E = len(ebh) - 1
        lst = []
        for e in range(E):
            cnt = ebh[e + 1] - ebh[e]
            for t in range(nt):
                for p in range(ebh[e], ebh[e + 1]):
                    lst.append(pr[p])
        lst = np.array(lst)
        g = 148
        nunits = np.array([len(lst[c::g]) for c in range(g)])
        mt = np.array([int(np.sum((lst[c::g] + 127) // 128)) for c in range(g)])
        rows = np.array([int(np.sum(lst[c::g])) for c in range(g)])
        e_ = (b - s) / 1e3
        print(f"    units {len(lst)}; per CTA units {nunits.min()}-{nunits.max()}, m-tiles {mt.min()}-{mt.max()}, "
              f"rows {rows.min()}-{rows.max()}")
        for k in sorted(set(mt)):
            sel = mt == k
            print(f"    m-tiles {k}: {sel.sum()} CTAs, end {e_[sel].min():.1f}-{e_[sel].max():.1f} us")
        A = np.stack([nunits, rows, np.ones(g)], 1)
        coef, *_ = np.linalg.lstsq(A, e_, rcond=None)
        print(f"    fit end ~ {coef[0]:.2f} us/unit + {coef[1]*128:.2f} us/128 rows + {coef[2]:.1f}; "
              f"resid std {np.std(e_ - A @ coef):.2f}")


if __name__ == "__main__":
    main()
