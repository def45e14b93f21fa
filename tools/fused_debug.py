"""Debug helper: which tokens does mp_ffn_fused get wrong (piece / tile position)?"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_ffn_fused_gpu import _segments, _weights, _fused, _reference, _zipf_route  # noqa
from paper_2605_11537_b200._dev import require_device

dev = require_device()
for (T, E, d, F, skew, div) in [(3000, 16, 768, 3072, 1.2, 96), (3000, 16, 768, 3072, 1.2, 10**9),
                                (256, 1, 768, 3072, 1.2, 10**9), (64, 1, 768, 3072, 1.2, 10**9),
                                (16, 1, 768, 3072, 1.2, 10**9), (128, 2, 768, 3072, 1.2, 10**9),
                                (2000, 8, 128, 512, 1.0, 10**9)]:
    rng = np.random.default_rng(T + d)
    route = _zipf_route(rng, T, E, skew, empty=E > 2)
    U, V, Ut, Vt = _weights(dev, E, d, F, seed=T + E)
    counts = np.bincount(route, minlength=E)
    cnt = np.maximum(1, counts // div).astype(np.int64)
    seg = _segments(dev, route, cnt)
    x = torch.randn(T, d, device=dev)
    y = x.clone()
    _fused(dev, x, y, d, F, E, Ut, Vt, seg)
    torch.cuda.synchronize()
    ref = _reference(x, route, U, V)
    err = ((y - x) - ref).abs().amax(dim=1) / ref.abs().max()
    bad = (err > 2e-3).nonzero().flatten().cpu().numpy()
    tor, prow, prows, eb = [t.cpu().numpy() for t in seg]
    row_of_tok = np.empty(T, dtype=np.int64)
    row_of_tok[tor] = np.arange(T)
    print(f"T={T} E={E} d={d} div={div}: bad tokens {len(bad)}/{T}, max err {err.max().item():.3e}")
    if len(bad):
        rows = np.sort(row_of_tok[bad])
        npieces = eb[-1]
        starts = prow[:npieces]
        lens = prows[:npieces]
        info = []
        for r in rows[:40]:
            p = np.nonzero((starts <= r) & (r < starts + lens))[0]
            p = p[0] if len(p) else -1
            info.append((int(r), int(p), int(r - starts[p]) if p >= 0 else -1, int(lens[p]) if p >= 0 else -1))
        print("  (row, piece, offset in piece, piece rows):", info)
        # per-column pattern of the first bad token
        t = bad[0]
        e_col = ((y - x) - ref)[t].abs()
        print("  first bad token", t, "bad dims:", (e_col > 2e-3 * ref.abs().max()).nonzero().flatten()[:20].tolist())
