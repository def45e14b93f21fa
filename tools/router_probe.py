"""Time the routing call (fused split-bf16 router + fp64 recheck) on the bench workload
(Switch-base-128 layer 0 router, a T=16384 synthetic batch)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402
from paper_2605_11537_b200.engine import PipelineConfig, SyntheticSwitch  # noqa: E402
from paper_2605_11537_b200.router_oracle import DeviceMoeLayer  # noqa: E402
from tools.gemm_probe import timeit  # noqa: E402


def main():
    dev = require_device()
    cfg = PipelineConfig()
    wl = SyntheticSwitch(cfg, dev)
    T, d, E = cfg.tokens, cfg.d_model, cfg.num_experts
    emb, _, routes = wl.batch(T)
    lay = DeviceMoeLayer.from_device(wl.router(0), torch.zeros(E, 256, d, device=dev, dtype=torch.bfloat16),
                                     torch.zeros(E, d, 256, device=dev, dtype=torch.bfloat16))
    route = torch.empty(T, dtype=torch.int32, device=dev)
    n = _lib.size_query("mp_router_workspace_bytes", T, d)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)

    def run():
        _lib.call("mp_route_top1_ex", ptr(emb), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                  ptr(route), ptr(ws), n, stream_ptr())

    us = timeit(run, iters=50)
    assert (route.long() == routes[0].long()).all()
    print(f"route_top1_ex: {us:.1f} us per call, host-launched (routing exact)")
    # device time: 20 calls captured in one CUDA graph (host launch overhead excluded)
    run()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(20):
            run()
    gus = timeit(g.replay, iters=10) / 20
    route.fill_(-1)
    g.replay()
    torch.cuda.synchronize()
    assert (route.long() == routes[0].long()).all()
    print(f"route_top1_ex: {gus:.1f} us per call in a CUDA graph (routing exact)")


if __name__ == "__main__":
    main()
