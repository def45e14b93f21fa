"""Time the fused expert FFN of one layer at config 3 (T=16k, E=128, d=768, F=3072) over the
engine's own replica pieces; print piece statistics. Env MP_FUSED_PREFETCH sets the L2 prefetch
distance. usage: python tools/fused_probe.py [capacity] [demand_unit] [replication] [ffn]"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 296
unit = int(sys.argv[2]) if len(sys.argv) > 2 else 128
rep = sys.argv[3] if len(sys.argv) > 3 else "on"
ffn = sys.argv[4] if len(sys.argv) > 4 else "fused"
layers = int(sys.argv[5]) if len(sys.argv) > 5 else 2
dev = require_device()
cfg = PipelineConfig(num_layers=layers, capacity=cap, demand_unit=unit, replication=rep, ffn=ffn)
t0 = time.time()
pipe = MoEPipeline(cfg, dev)
x0, _, _ = pipe.wl.batch(cfg.tokens)
x = x0.clone()
pipe.step(x)
x = x0.clone()
pipe.step(x)  # second batch: warm residency
torch.cuda.synchronize()
l = 0
eb = pipe.exp_begin[l].cpu().numpy()
npieces = int(eb[-1])
rows = pipe.piece_rows[l, :npieces].cpu().numpy()
NT = 64
tiles = int(np.ceil(rows[rows > 0] / NT).sum())
print(f"cap={cap} unit={unit} rep={rep} ffn={pipe.cfg.ffn}: pieces {npieces} (nonempty {(rows > 0).sum()}), "
      f"tiles {tiles}, max piece rows {rows.max()}, setup {time.time() - t0:.1f}s")
T, d, F, E = cfg.tokens, cfg.d_model, cfg.d_ff, cfg.num_experts
lay = pipe.layers[l]
sp = stream_ptr()


def run():
    if pipe.cfg.ffn == "fused":
        _lib.call("mp_ffn_fused", ptr(x), T, d, F, E, ptr(lay.U), ptr(lay.V), 0, ptr(pipe.tok_of_row[l]),
                  ptr(pipe.piece_row[l]), ptr(pipe.piece_rows[l]), ptr(pipe.exp_begin[l]), ptr(pipe.ws_ffn),
                  pipe.ws_ffn_n, sp)
    else:
        flags = lay.tiled | (2 if pipe.cfg.ffn == "pair" else 0)
        _lib.call("mp_ffn_up", T, d, F, E, ptr(lay.U), flags, ptr(pipe.piece_row[l]), ptr(pipe.piece_rows[l]),
                  ptr(pipe.exp_begin[l]), ptr(pipe.ws_ffn), pipe.ws_ffn_n, sp)
        _lib.call("mp_ffn_down", ptr(x), T, d, F, E, ptr(lay.V), flags, ptr(pipe.tok_of_row[l]),
                  ptr(pipe.piece_row[l]), ptr(pipe.piece_rows[l]), ptr(pipe.exp_begin[l]), ptr(pipe.ws_ffn),
                  pipe.ws_ffn_n, sp)


_lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(pipe.tok_of_row[l]), ptr(pipe.ws_ffn), pipe.ws_ffn_n, sp)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
for _ in range(3):
    run()
times = []
for _ in range(10):
    flush.zero_()  # evict the layer's weights from L2 (a step streams 14.5 GB between visits)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    run()
    b.record()
    torch.cuda.synchronize()
    times.append(a.elapsed_time(b) * 1e3)
touched = int((eb[1:] > eb[:-1]).sum())
alg = touched * 4 * d * F + T * 10 * d
med = float(np.median(times))
print(f"  FFN {med:.1f} us (min {min(times):.1f}); alg bytes {alg / 1e9:.3f} GB -> {alg / med / 1e3:.0f} GB/s "
      f"= {alg / med / 1e3 / 6529.4:.3f} of HBM")
import os  # noqa: E402
if os.environ.get("MP_FUSED_DEBUG"):
    import ctypes
    buf = (ctypes.c_ulonglong * (148 * 16))()
    _lib.call("mp_debug_fused_waits", ctypes.addressof(buf), 148 * 16)
    w = np.array(buf[:], dtype=np.float64).reshape(148, 16)
    names = ["prod-empty", "prod-xempty", "mma-full-G1", "mma-full-G2", "mma-hfull", "mma-t1empty", "mma-xfull",
             "epi-t1full", "epi-hempty", "epi-d2full", "sched-want", "epi-life"]
    life = w[:, 11]
    for k, nme in enumerate(names):
        print(f"  {nme:12s} mean {w[:, k].mean() / 1965:8.1f} us  ({w[:, k].mean() / life.mean():.2f} of life)")
