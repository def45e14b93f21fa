"""CUDA expert-parallel kernels on one GPU: the plan for every rank of a simulated
G-GPU job (planning is per rank and needs no peers) must equal the oracle plan;
the G = 1 expert-parallel forward must equal the single-device forward bitwise."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from oracle.ep_oracle import ep_plan  # noqa: E402
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402


@pytest.mark.parametrize("G,E,T", [(4, 16, 500), (8, 128, 2048), (2, 7, 33), (3, 256, 4000)])
def test_ep_plan_matches_oracle_for_every_rank(G, E, T):
    dev = require_device()
    rng = np.random.default_rng(G * 100 + E)
    w = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    routes = [rng.choice(E, size=T, p=w / w.sum()) for _ in range(G)]
    C = np.stack([np.bincount(r, minlength=E) for r in routes]).astype(np.int32)
    res0 = rng.integers(0, 4, size=E).astype(np.int32)
    max_slots = int(res0.sum()) + E + 1
    i32 = dict(dtype=torch.int32, device=dev)
    Cd = torch.from_numpy(C).to(dev)
    for r in range(G):
        ref = ep_plan(routes[r], C, res0.astype(np.int64).copy(), r)
        res = torch.from_numpy(res0.copy()).to(dev)
        sc, rc, nl = torch.empty(G, **i32), torch.empty(G, **i32), torch.empty(1, **i32)
        sp = torch.empty(T, **i32)
        pn = max_slots + (G * T + 127) // 128
        prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
        n = _lib.size_query("mp_ep_workspace_bytes", G, T, E, max_slots)
        ws = torch.empty(n, dtype=torch.uint8, device=dev)
        route = torch.from_numpy(routes[r].astype(np.int32)).to(dev)
        _lib.call("mp_ep_plan", ptr(route), T, ptr(Cd), G, E, r, max_slots, 1, ptr(res), ptr(sc), ptr(rc), ptr(nl),
                  ptr(sp), ptr(prow), ptr(prows), ptr(eb), ptr(ws), n, stream_ptr())
        rol = torch.empty(G * T, **i32)
        _lib.call("mp_ep_recv_layout", G, T, E, r, max_slots, None, ptr(rol), ptr(ws), n, stream_ptr())
        torch.cuda.synchronize()
        assert sc.cpu().tolist() == ref["send_counts"].tolist()
        assert rc.cpu().tolist() == ref["recv_counts"].tolist()
        assert int(nl.item()) == ref["n_local"]
        assert (sp.cpu().numpy() == ref["send_pos"]).all()
        assert (rol[: ref["n_local"]].cpu().numpy() == ref["recv_of_local"]).all()
        ebh, prow_h, prows_h = eb.cpu().numpy(), prow.cpu().numpy(), prows.cpu().numpy()
        got = [(e, int(prow_h[p]), int(prows_h[p])) for e in range(E) for p in range(ebh[e], ebh[e + 1])]
        assert got == ref["pieces"]


def test_expert_parallel_single_rank_equals_dense_forward():
    from paper_2605_11537_b200.ep import CudaEpKernels, ExpertParallelMoE
    from paper_2605_11537_b200.router_oracle import ToyMoeParams, _device_moe, _run_layers_device

    dev = require_device()
    rng = np.random.default_rng(1)
    L, E, d, F, T = 3, 16, 256, 512, 3000
    params = ToyMoeParams(rng.normal(size=(L, E, d)).astype(np.float32),
                          (rng.normal(size=(L, E, F, d)) / 16).astype(np.float32),
                          (rng.normal(size=(L, E, d, F)) / 23).astype(np.float32))
    dm = _device_moe(params, dev)
    x0 = torch.from_numpy(rng.normal(size=(T, d)).astype(np.float32)).to(dev)
    x_ref = x0.clone()
    _run_layers_device(x_ref, dm)
    for lay in dm.layers:  # EP path uses pre-tiled weights
        u2, v2 = lay.U.clone(), lay.V.clone()
        _lib.call("mp_tile_kmajor", ptr(u2), ptr(lay.U), E, F, d, _lib.size_query("mp_ffn_up_bn", F), stream_ptr())
        _lib.call("mp_tile_kmajor", ptr(v2), ptr(lay.V), E, d, F, _lib.size_query("mp_ffn_down_bn", d), stream_ptr())
        lay.tiled = 1
    k = CudaEpKernels(dm.layers, T, 1, 0, max_slots=4 * E)
    ep = ExpertParallelMoE(k, L, E)
    x_ep = x0.clone()
    ep.forward(x_ep)
    torch.cuda.synchronize()
    assert torch.equal(x_ep, x_ref)


@pytest.mark.parametrize("G", [2, 3, 4])
def test_token_sharded_sru_equals_whole_sequence(G):
    """the G ranks' token ranges are one SRU sequence. Each simulated rank
    projects its rows, reduces them to one carry map, the maps are 'all-gathered' (here:
    stacked), folded into each rank's carry-in, and the replay from it must reproduce the
    unsharded layer (fp32 carry re-association only)."""
    dev = require_device()
    T, d = 256 * G * 2, 256
    g = torch.Generator(device=dev).manual_seed(G)
    x = torch.randn(T, d, device=dev, generator=g) * 0.5
    xb = x.bfloat16()
    w = (torch.randn(3 * d, d, device=dev, generator=g) / d ** 0.5).bfloat16()
    b = torch.randn(3 * d, device=dev, generator=g) * 0.1
    nf = torch.zeros(1, dtype=torch.int32, device=dev)
    n = _lib.size_query("mp_sru_workspace_bytes", T, d)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    h_ref = torch.empty(T, d, device=dev)
    h16 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    _lib.call("mp_sru_layer", ptr(xb), ptr(x), ptr(w), ptr(b), T, d, None, ptr(h_ref), ptr(h16), None, ptr(nf),
              ptr(ws), n, stream_ptr())
    Tg = T // G
    ng = _lib.size_query("mp_sru_workspace_bytes", Tg, d)
    wss = [torch.empty(ng, dtype=torch.uint8, device=dev) for _ in range(G)]
    tots = torch.empty(G, 2 * d, device=dev)
    for r in range(G):  # every rank: project + whole-range map
        rows = slice(r * Tg, (r + 1) * Tg)
        _lib.call("mp_sru_project", ptr(xb[rows]), ptr(w), ptr(b), Tg, d, ptr(wss[r]), ng, stream_ptr())
        _lib.call("mp_sru_scan_total", Tg, d, ptr(tots[r]), ptr(wss[r]), ng, stream_ptr())
    h = torch.empty(T, d, device=dev)
    hb = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    cin = torch.empty(d, device=dev)
    for r in range(G):  # after the all-gather: fold + replay
        rows = slice(r * Tg, (r + 1) * Tg)
        _lib.call("mp_sru_fold_carry", ptr(tots), r, d, None, ptr(cin), stream_ptr())
        _lib.call("mp_sru_scan_finish", ptr(x[rows]), Tg, d, ptr(cin), ptr(h[rows]), ptr(hb[rows]), None, ptr(nf),
                  ptr(wss[r]), ng, stream_ptr())
    torch.cuda.synchronize()
    rel = ((h - h_ref).abs().max() / h_ref.abs().max()).item()
    assert rel < 1e-5, rel
    assert int(nf.item()) == 0


def test_peer_memory_tables_map_another_process(tmp_path):
    """ep.PeerMemory across two processes on this GPU (CUDA IPC through torch's storage sharing,
    gloo for the handles): each rank's table entry for the other rank addresses that rank's
    buffer view (storage offset included) -- read back with a plain gather kernel."""
    import socket
    import subprocess
    import sys
    from pathlib import Path

    require_device()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    worker = Path(__file__).resolve().parent / "peer_worker.py"
    out = tmp_path / "peer"
    procs = [subprocess.Popen([sys.executable, str(worker), str(r), "2", str(port), str(out)]) for r in range(2)]
    try:
        for p in procs:
            assert p.wait(timeout=240) == 0
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert [Path(f"{out}.{r}").read_text() for r in range(2)] == ["ok", "ok"]


def test_peer_memory_ep_across_two_processes(tmp_path):
    """The peer-memory EP data path between two processes on this GPU through real CUDA IPC
    peer tables (receive rows and residual streams of the other process), host barriers in
    place of the device barriers: each rank's shard equals the single-device forward."""
    import socket
    import subprocess
    import sys
    from pathlib import Path

    require_device()
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    worker = Path(__file__).resolve().parent / "peer_ep_worker.py"
    out = tmp_path / "pep"
    procs = [subprocess.Popen([sys.executable, str(worker), str(r), "2", str(port), str(out)]) for r in range(2)]
    try:
        for p in procs:
            assert p.wait(timeout=300) == 0
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert [Path(f"{out}.{r}").read_text() for r in range(2)] == ["ok", "ok"]
