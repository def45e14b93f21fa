"""Would a hybrid grouped GEMM (CTA pairs for the pieces of hot experts, single CTAs for cold
experts) beat single CTAs everywhere at config 3? Times GEMM1 + GEMM2 on a Zipf-1.2 routing:
(a) all tokens, single-CTA kernels; (b) hot-expert tokens through the pair kernels + the
cold-expert tokens through the single-CTA kernels (two launches each)."""
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
    hot_min = int(sys.argv[1]) if len(sys.argv) > 1 else 256  # rows for an expert to count as hot
    U0 = (torch.randn(E * F, d, device=dev) / 30).bfloat16()
    V0 = (torch.randn(E * d, F, device=dev) / 55).bfloat16()
    U, V1, V2 = torch.empty_like(U0), torch.empty_like(V0), torch.empty_like(V0)
    _lib.call("mp_tile_kmajor", ptr(U0), ptr(U), E, F, d, 256, stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(V0), ptr(V1), E, d, F, _lib.size_query("mp_ffn_down_bn", d), stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(V0), ptr(V2), E, d, F, 256, stream_ptr())
    rng = np.random.default_rng(0)
    w = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    route = rng.choice(E, size=T, p=w / w.sum())
    counts = np.bincount(route, minlength=E)
    hot = counts >= hot_min
    i32 = dict(dtype=torch.int32, device=dev)

    def prepare(mask, split):
        sel = mask[route]
        r = route[sel].astype(np.int32)
        n = len(r)
        rt = torch.from_numpy(r).to(dev)
        se = torch.arange(E, dtype=torch.int32, device=dev)
        pn = 2 * (E + n // 128 + 1)
        tor, prow, prows, eb = torch.empty(n, **i32), torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
        nb = _lib.size_query("mp_segments_workspace_bytes", n, E)
        sws = torch.empty(nb, dtype=torch.uint8, device=dev)
        _lib.call("mp_segments_from_slots", ptr(rt), ptr(se), n, E, E, split, ptr(tor), ptr(prow), ptr(prows), ptr(eb),
                  ptr(sws), nb, stream_ptr())
        fb = _lib.size_query("mp_ffn_workspace_bytes", n, d, F)
        ws = torch.empty(fb, dtype=torch.uint8, device=dev)
        x = torch.randn(n, d, device=dev)
        _lib.call("mp_ffn_gather", ptr(x), n, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())
        y = x.clone()
        return dict(n=n, tor=tor, prow=prow, prows=prows, eb=eb, ws=ws, fb=fb, y=y)

    def gemms(s, flags, v):
        _lib.call("mp_ffn_up", s["n"], d, F, E, ptr(U), flags, ptr(s["prow"]), ptr(s["prows"]), ptr(s["eb"]),
                  ptr(s["ws"]), s["fb"], stream_ptr())
        _lib.call("mp_ffn_down", ptr(s["y"]), s["n"], d, F, E, ptr(v), flags, ptr(s["tor"]), ptr(s["prow"]),
                  ptr(s["prows"]), ptr(s["eb"]), ptr(s["ws"]), s["fb"], stream_ptr())

    all_s = prepare(np.ones(E, dtype=bool), 1)
    hot_s = prepare(hot, 3)
    cold_s = prepare(~hot, 1)
    t_all = timeit(lambda: gemms(all_s, 1, V1), iters=10)
    t_hyb = timeit(lambda: (gemms(hot_s, 3, V2), gemms(cold_s, 1, V1)), iters=10)
    t_hot1 = timeit(lambda: gemms(hot_s, 1, V1), iters=10)
    t_hot2 = timeit(lambda: gemms(hot_s, 3, V2), iters=10)
    t_cold = timeit(lambda: gemms(cold_s, 1, V1), iters=10)
    print(f"hot >= {hot_min} rows: {hot.sum()} experts, {hot_s['n']} of {T} tokens")
    print(f"single everywhere {t_all:.1f} us | hybrid {t_hyb:.1f} us (hot pair {t_hot2:.1f} vs single {t_hot1:.1f}, "
          f"cold single {t_cold:.1f})")


if __name__ == "__main__":
    main()
