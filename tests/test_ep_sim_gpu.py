"""Expert parallelism over a SIMULATED G-GPU job on one device.

Every rank's CUDA kernels run on this GPU: route -> counts -> plan -> pack -> (all-to-all
emulated by device copies in NCCL's layout) -> receive layout -> grouped GEMMs -> (reverse
all-to-all) -> combine. Ranks never wait on one another inside a kernel; the host plays the
collectives between the per-rank launches. The result over the G token shards must equal the
single-device forward of the whole batch bit for bit, with and without replicas, at the
Switch-base widths and for both V tilings (single-CTA 192-column and CTA-pair 256-column)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402


def _params(L, E, d, F, seed):
    from paper_2605_11537_b200.router_oracle import ToyMoeParams
    rng = np.random.default_rng(seed)
    return ToyMoeParams(rng.normal(size=(L, E, d)).astype(np.float32),
                        (rng.normal(size=(L, E, F, d)) / np.sqrt(d)).astype(np.float32),
                        (rng.normal(size=(L, E, d, F)) / np.sqrt(F)).astype(np.float32))


def _tile(dm, E, d, F, vbn):
    for lay in dm.layers:
        u2, v2 = lay.U.clone(), lay.V.clone()
        _lib.call("mp_tile_kmajor", ptr(u2), ptr(lay.U), E, F, d, _lib.size_query("mp_ffn_up_bn", F), stream_ptr())
        _lib.call("mp_tile_kmajor", ptr(v2), ptr(lay.V), E, d, F, vbn, stream_ptr())
        lay.tiled = 1
        lay.vbn = vbn


def _a2a(chunks_by_src, counts, dst_bufs):
    """NCCL all_to_all_single layout: rank r receives, in source order, the block every
    source g sends it (source g's send buffer is destination-major)."""
    G = len(chunks_by_src)
    for r in range(G):
        parts = []
        for g in range(G):
            displ = sum(counts[g][:r])
            parts.append(chunks_by_src[g][displ:displ + counts[g][r]])
        if parts:
            dst_bufs[r].copy_(torch.cat(parts))


def _simulate(ks, xs, res, L):
    G = len(ks)
    for l in range(L):
        routes = [k.route(x, l) for k, x in zip(ks, xs)]
        C = torch.stack([k.counts(r).clone() for k, r in zip(ks, routes)])
        plans = [k.plan(r, C, res[g][l], x) for g, (k, r, x) in enumerate(zip(ks, routes, xs))]
        sends = [k.pack(x, p, sum(p.send_counts)) for k, x, p in zip(ks, xs, plans)]
        recvs = [k.recv_buffer(sum(p.recv_counts)) for k, p in zip(ks, plans)]
        _a2a(sends, [p.send_counts for p in plans], recvs)
        ys = [k.expert_ffn(rb, p, l) for k, rb, p in zip(ks, recvs, plans)]
        backs = [k.back_buffer(sum(p.send_counts)) for k, p in zip(ks, plans)]
        _a2a(ys, [p.recv_counts for p in plans], backs)
        for k, x, yb, p in zip(ks, xs, backs, plans):
            k.combine(x, yb, p)
    return plans


@pytest.mark.parametrize("G,E,d,F,T,vbn,replicas", [
    (2, 16, 256, 512, 700, None, False), (4, 16, 256, 512, 500, None, True), (8, 32, 256, 512, 300, None, True),
    (2, 16, 768, 3072, 600, None, True), (4, 8, 768, 3072, 300, 256, True), (3, 12, 768, 3072, 257, None, False)])
def test_simulated_ep_equals_single_device(G, E, d, F, T, vbn, replicas):
    from paper_2605_11537_b200.ep import CudaEpKernels
    from paper_2605_11537_b200.router_oracle import _device_moe, _run_layers_device

    dev = require_device()
    L = 2
    params = _params(L, E, d, F, seed=G * 10 + E + d)
    rng = np.random.default_rng(G)
    # Zipf-skewed tokens: rows near one router row route to that expert
    pop = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    e0 = rng.choice(E, size=G * T, p=pop / pop.sum())
    x0 = (params.router_weights[0][e0] * 0.05 + rng.normal(size=(G * T, d)) * 0.5).astype(np.float32)
    dm_ref = _device_moe(params, dev)
    x_ref = torch.from_numpy(x0).to(dev)
    _run_layers_device(x_ref, dm_ref)  # dense single-device forward of the whole batch
    dm = _device_moe(params, dev)
    _tile(dm, E, d, F, vbn or _lib.size_query("mp_ffn_down_bn", d))
    res0 = (rng.integers(0, 4, size=(L, E)) if replicas else np.zeros((L, E))).astype(np.int32)
    capacity = int(res0.sum(1).max()) + E
    ks = [CudaEpKernels(dm.layers, T, G, r, G * capacity + E) for r in range(G)]
    res = [torch.from_numpy(res0.copy()).to(dev) for _ in range(G)]
    xs = [torch.from_numpy(x0[r * T:(r + 1) * T].copy()).to(dev) for r in range(G)]
    plans = _simulate(ks, xs, res, L)
    torch.cuda.synchronize()
    out = torch.cat(xs)
    assert torch.equal(out, x_ref)
    for g in range(1, G):  # every rank holds the same residency state
        assert torch.equal(res[g], res[0])
    # row budget: the slot list is cut into G blocks of equal rows
    rows = [sum(p.recv_counts) for p in plans]
    assert max(rows) - min(rows) <= max(1, (G * T) // 2), rows


def test_ep_plan_over_capacity_raises_before_collectives():
    """More execution slots than max_slots: mp_ep_plan reports it through the sizes the host
    reads (num_local_rows = -1, zero counts) and the host raises instead of issuing an
    all-to-all with stale split sizes."""
    from paper_2605_11537_b200.ep import CudaEpKernels
    from paper_2605_11537_b200.errors import ConfigurationError
    from paper_2605_11537_b200.router_oracle import _device_moe

    dev = require_device()
    E, d, F, T = 8, 256, 512, 200
    dm = _device_moe(_params(1, E, d, F, seed=3), dev)
    k = CudaEpKernels(dm.layers, T, 2, 0, max_slots=E)
    route = torch.randint(0, E, (T,), dtype=torch.int32, device=dev)
    C = torch.stack([k.counts(route).clone(), k.counts(route).clone()])
    res = torch.full((E,), 3, dtype=torch.int32, device=dev)  # 24 slots > max_slots = 8
    with pytest.raises(ConfigurationError):
        k.plan(route, C, res)


@pytest.mark.parametrize("G,E,d,F,T,replicas", [(2, 16, 256, 512, 700, True), (4, 16, 768, 3072, 300, True),
                                                 (8, 32, 256, 512, 300, False)])
def test_simulated_fixed_split_ep_equals_single_device(G, E, d, F, T, replicas):
    """Fixed-split dispatch (static all-to-all splits of peer_cap rows per (source, destination)
    block, graph-capturable): same bits as the single-device forward, no overflow."""
    from paper_2605_11537_b200.ep import CudaEpKernels
    from paper_2605_11537_b200.router_oracle import _device_moe, _run_layers_device

    dev = require_device()
    L = 2
    params = _params(L, E, d, F, seed=7 * G + E)
    rng = np.random.default_rng(100 + G)
    pop = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    e0 = rng.choice(E, size=G * T, p=pop / pop.sum())
    x0 = (params.router_weights[0][e0] * 0.05 + rng.normal(size=(G * T, d)) * 0.5).astype(np.float32)
    x_ref = torch.from_numpy(x0).to(dev)
    _run_layers_device(x_ref, _device_moe(params, dev))
    dm = _device_moe(params, dev)
    _tile(dm, E, d, F, _lib.size_query("mp_ffn_down_bn", d))
    res0 = (rng.integers(0, 4, size=(L, E)) if replicas else np.zeros((L, E))).astype(np.int32)
    capacity = int(res0.sum(1).max()) + E
    cap = T if G == 1 else -(-2 * T // G)
    ks = [CudaEpKernels(dm.layers, T, G, r, G * capacity + E, peer_cap=cap) for r in range(G)]
    res = [torch.from_numpy(res0.copy()).to(dev) for _ in range(G)]
    xs = [torch.from_numpy(x0[r * T:(r + 1) * T].copy()).to(dev) for r in range(G)]
    _simulate(ks, xs, res, L)
    torch.cuda.synchronize()
    assert all(int(k.overflow.item()) == 0 for k in ks)
    assert torch.equal(torch.cat(xs), x_ref)


def test_simulated_fixed_split_overflow_is_a_flagged_no_op():
    """A fixed split too small for the layer: EVERY rank flags the overflow (the decision comes
    from the all-gathered counts, so the ranks agree and re-run together) and the layer leaves
    every rank's residual stream untouched."""
    from paper_2605_11537_b200.ep import CudaEpKernels
    from paper_2605_11537_b200.router_oracle import _device_moe

    dev = require_device()
    G, E, d, F, T = 4, 16, 256, 512, 400
    params = _params(1, E, d, F, seed=11)
    dm = _device_moe(params, dev)
    _tile(dm, E, d, F, _lib.size_query("mp_ffn_down_bn", d))
    rng = np.random.default_rng(5)
    x0 = rng.normal(size=(G * T, d)).astype(np.float32)
    ks = [CudaEpKernels(dm.layers, T, G, r, G * (E + 8) + E, peer_cap=16) for r in range(G)]
    res = [torch.zeros(1, E, dtype=torch.int32, device=dev) for _ in range(G)]
    xs = [torch.from_numpy(x0[r * T:(r + 1) * T].copy()).to(dev) for r in range(G)]
    _simulate(ks, xs, res, 1)
    torch.cuda.synchronize()
    assert all(int(k.overflow.item()) == 1 for k in ks)
    assert torch.equal(torch.cat(xs).cpu(), torch.from_numpy(x0))


@pytest.mark.parametrize("G,E,d,F,T,replicas", [(2, 16, 256, 512, 700, True), (4, 16, 768, 3072, 300, True),
                                                 (8, 32, 256, 512, 300, False)])
def test_simulated_peer_memory_ep_equals_single_device(G, E, d, F, T, replicas):
    """Peer-memory dispatch / combine (no all-to-all): every rank writes its rows into the
    destinations' receive blocks and the destinations' GEMM2 epilogues add the results into the
    home streams through peer address tables -- here G ranks' buffers on one device, the ranks'
    kernels issued one after another (no device barrier: nothing waits inside a kernel). Same
    bits as the single-device forward."""
    from paper_2605_11537_b200.ep import CudaEpKernels
    from paper_2605_11537_b200.router_oracle import _device_moe, _run_layers_device

    dev = require_device()
    L = 2
    params = _params(L, E, d, F, seed=13 * G + E)
    rng = np.random.default_rng(200 + G)
    pop = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
    e0 = rng.choice(E, size=G * T, p=pop / pop.sum())
    x0 = (params.router_weights[0][e0] * 0.05 + rng.normal(size=(G * T, d)) * 0.5).astype(np.float32)
    x_ref = torch.from_numpy(x0).to(dev)
    _run_layers_device(x_ref, _device_moe(params, dev))
    dm = _device_moe(params, dev)
    _tile(dm, E, d, F, _lib.size_query("mp_ffn_down_bn", d))
    res0 = (rng.integers(0, 4, size=(L, E)) if replicas else np.zeros((L, E))).astype(np.int32)
    capacity = int(res0.sum(1).max()) + E
    cap = -(-2 * T // G)
    ks = [CudaEpKernels(dm.layers, T, G, r, G * capacity + E, peer_cap=cap, p2p=True) for r in range(G)]
    res = [torch.from_numpy(res0.copy()).to(dev) for _ in range(G)]
    xs = [torch.from_numpy(x0[r * T:(r + 1) * T].copy()).to(dev) for r in range(G)]
    table = lambda ts: torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64, device=dev)
    t_recv, t_tok, t_flags, t_x, t_C = (table([k.recvbuf for k in ks]), table([k.recv_tok for k in ks]),
                                        table([k.flags for k in ks]), table(xs), table([k.C_all for k in ks]))
    for k, x in zip(ks, xs):
        k.set_peers(t_recv, t_tok, t_flags, t_C)
        k.register_stream(x, t_x)
    for l in range(L):
        routes = [k.route(x, l) for k, x in zip(ks, xs)]
        for k, r in zip(ks, routes):  # the counts all-gather by peer stores (no barrier needed here)
            k.allgather_counts_peer(k.counts(r), barrier=False)
        C = torch.stack([k.counts(r).clone() for k, r in zip(ks, routes)])
        assert all(torch.equal(k.C_all, C) for k in ks)
        plans = [k.plan(r, k.C_all, res[g][l]) for g, (k, r) in enumerate(zip(ks, routes))]
        for k, x, p in zip(ks, xs, plans):
            k.dispatch_peer(x, p)
        for k, p in zip(ks, plans):
            k.expert_ffn_peer(p, l)
    torch.cuda.synchronize()
    assert all(int(k.overflow.item()) == 0 for k in ks)
    assert torch.equal(torch.cat(xs), x_ref)
