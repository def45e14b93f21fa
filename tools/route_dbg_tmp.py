import sys, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2605_11537_b200 import _lib
from paper_2605_11537_b200._dev import require_device, ptr, stream_ptr
from paper_2605_11537_b200.router_oracle import ToyMoeParams, _device_moe
dev = require_device()
E, d, T = 16, 768, 5000
rng = np.random.default_rng(1)
W = rng.normal(size=(1, E, d)).astype(np.float32)
params = ToyMoeParams(W, np.zeros((1, E, 256, d), np.float32), np.zeros((1, E, d, 256), np.float32))
lay = _device_moe(params, dev).layers[0]
e0 = rng.choice(E, size=T)
x = torch.from_numpy((W[0][e0] * 0.05 + rng.normal(size=(T, d)) * 0.5).astype(np.float32)).to(dev)
Wd = torch.from_numpy(W[0]).to(dev).double()
lg = x.double() @ Wd.T
rb = _lib.size_query("mp_router_workspace_bytes", T, d)
ws = torch.empty(rb, dtype=torch.uint8, device=dev)
route = torch.empty(T, dtype=torch.int32, device=dev)
_lib.call("mp_route_top1_ex", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
          ptr(route), ptr(ws), rb, stream_ptr())
torch.cuda.synchronize()
buf = np.zeros(T * E, np.float32)
_lib.call("mp_debug_router_logits", buf.ctypes.data, T * E)
tc = torch.from_numpy(buf.reshape(T, E)).to(dev).double()
err = (tc - lg).abs().amax(1)
bad = (err > 1e-2).nonzero().flatten()
print("tokens with logit error > 1e-2:", len(bad), "of", T, " max err", err.max().item())
print("bad tokens (first 20):", bad[:20].tolist())
print("rows within tile of bad:", (bad % 128)[:40].tolist())
print("tiles of bad:", sorted(set((bad // 128).tolist()))[:30])
# per-k-block decomposition of the error for the first bad tokens
xk = x.double().view(T, d // 64, 64)
Wk = Wd.view(E, d // 64, 64)
contrib = torch.einsum("tkc,ekc->tke", xk, Wk)  # (T, nkb, E)
for t in bad[:6].tolist():
    e_vec = tc[t] - lg[t]
    # error = missing kb? duplicated kb? stale kb from another token?
    best = None
    for kb in range(d // 64):
        for sgn in (-1, 1):
            r = (e_vec - sgn * contrib[t, kb]).abs().max().item()
            if best is None or r < best[0]:
                best = (r, kb, sgn)
    # other-token hypothesis: tc = lg - contrib[t,kb] + contrib[t2,kb]
    diff = e_vec[None, None, :] + contrib[t][None, :, :] - contrib  # (T, nkb, E)
    res = diff.abs().amax(2)
    v, idx = res.view(-1).min(0)
    t2, kb2 = divmod(int(idx), d // 64)
    print(f"token {t} (row {t % 128}): |err| {e_vec.abs().max().item():.3f}; best +-kb fit residual {best[0]:.4f} "
          f"kb={best[1]} sgn={best[2]}; swap fit: kb {kb2} from token {t2} (row {t2 % 128}, tile {t2 // 128}) residual {v.item():.4f}")
