"""Distribution of the grouped-FFN max-norm error vs an fp32 torch reference over seeds (test margin check)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402


def main():
    dev = require_device()
    T, E, d, F = 1500, 10, 128, 256
    rng = np.random.default_rng(3)
    route = rng.choice(E, size=T, p=np.array([0.5] + [0.5 / (E - 1)] * (E - 1))).astype(np.int32)
    rt = torch.from_numpy(route).to(dev)
    se = torch.arange(E, dtype=torch.int32, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    tor = torch.empty(T, **i32)
    pn = E + T // 128 + 1
    prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
    nb = _lib.size_query("mp_segments_workspace_bytes", T, E)
    sws = torch.empty(nb, dtype=torch.uint8, device=dev)
    _lib.call("mp_segments_from_slots", ptr(rt), ptr(se), T, E, E, 0, ptr(tor), ptr(prow), ptr(prows), ptr(eb),
              ptr(sws), nb, stream_ptr())
    errs = []
    for seed in range(40):
        g = torch.Generator(device=dev).manual_seed(seed)
        U = torch.randn(E, F, d, device=dev, generator=g) / np.sqrt(d)
        V = torch.randn(E, d, F, device=dev, generator=g) / np.sqrt(F)
        x = torch.randn(T, d, device=dev, generator=g)
        x0 = x.clone()
        Ub, Vb = U.bfloat16().contiguous(), V.bfloat16().contiguous()
        fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
        fws = torch.empty(fb, dtype=torch.uint8, device=dev)
        _lib.call("mp_moe_ffn", ptr(x), ptr(x), T, d, F, E, ptr(Ub), ptr(Vb), ptr(tor), ptr(prow), ptr(prows), ptr(eb),
                  ptr(fws), fb, stream_ptr())
        xb = x0.bfloat16().float()
        ref = x0.clone()
        rl = rt.long()
        for e in range(E):
            m = rl == e
            hid = (xb[m] @ Ub[e].float().T).relu().bfloat16().float()
            ref[m] += hid @ Vb[e].float().T
        a, b = (x - x0).double(), (ref - x0).double()
        errs.append(float((a - b).abs().max() / b.abs().max()))
    print("max rel err over seeds: median %.2e  max %.2e" % (np.median(errs), max(errs)))


if __name__ == "__main__":
    main()
