"""Device-resident engine (MoEPipeline) on a small Switch-like workload: routing (fused
split-bf16 router) must be the workload's exact float64 routing at every layer, and the
residual stream must not depend on how replicas/tiles are laid out (replication on,
split, off and the CTA-pair FFN kernels give the same bits)."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(replication="on", ffn="two", full=False):
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=4, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=3,
                         capacity=64, ffn=ffn, replication=replication, seed=3)
    pipe = MoEPipeline(cfg)
    emb, _, oracle_routes = pipe.wl.batch(cfg.tokens)
    x = emb.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipe.step(x)
    torch.cuda.synchronize()
    if full:
        return pipe
    return x, pipe.route.clone(), oracle_routes


def test_engine_routing_exact_and_layout_independent():
    x_on, r_on, oracle = _run("on")
    assert (r_on.long() == oracle.long()).all()
    for rep, ffn in (("split", "two"), ("off", "two"), ("on", "pair"), ("off", "pair")):
        x, r, _ = _run(rep, ffn)
        assert torch.equal(r, r_on), (rep, ffn)
        assert torch.equal(x, x_on), (rep, ffn)


def test_expert_parallel_step_through_nccl_single_rank():
    """The expert-parallel step with every collective issued through a real NCCL process group
    (world size 1: all-gather of counts and of the sharded SRU carry maps, variable all-to-all
    dispatch and combine) == the single-device step, bit for bit."""
    import socket

    import torch.distributed as dist

    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=3,
                             capacity=64, seed=5)
        a = MoEPipeline(cfg)
        emb, _, oracle = a.wl.batch(cfg.tokens)
        xa = emb.clone()
        a.step(xa)
        b = MoEPipeline(cfg)
        b.enable_expert_parallel()
        b.force_collectives = True
        xb = emb.clone()
        for _ in range(2):  # the second step reuses the residency planned by the first
            xb.copy_(emb)
            b.step(xb)
        torch.cuda.synchronize()
        assert torch.equal(b.ep.last_route.long(), oracle[-1].long())
        assert torch.equal(xa, xb)
    finally:
        dist.destroy_process_group()


def test_engine_step_matches_cpu_oracle_moe_forward():
    """The engine's whole step (predictor, plan, placement, 4 MoE layers on the device) against
    the CPU oracle's MoE forward (oracle/moesim_oracle.py, reference router_oracle.py:119-135) on
    the SAME embeddings and weights: the residual stream within 1e-2 max-norm relative (bf16
    operands vs fp32), routing decisions equal."""
    import numpy as np

    from oracle import moesim_oracle as O
    from paper_2605_11537_b200 import _lib
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=4, num_experts=32, d_model=256, d_ff=512, tokens=2048, sru_layers=3,
                         capacity=64, seed=11)
    pipe = MoEPipeline(cfg)
    emb, _, _ = pipe.wl.batch(cfg.tokens)
    x = emb.clone()
    pipe.step(x)
    torch.cuda.synchronize()
    E, d, F = cfg.num_experts, cfg.d_model, cfg.d_ff

    def untile(t, N, K, bn):  # mp_tile_kmajor layout [E][N/bn][K/64][bn][64] -> [E][N][K]
        return t.view(E, N // bn, K // 64, bn, 64).permute(0, 1, 3, 2, 4).reshape(E, N, K)

    ubn = _lib.size_query("mp_ffn_up_bn", F)
    vbn = _lib.size_query("mp_ffn_down_bn", d)
    router = np.stack([pipe.wl.router(l).cpu().numpy() for l in range(cfg.num_layers)]).astype(np.float32)
    eu = np.stack([untile(lay.U, F, d, ubn).float().cpu().numpy() for lay in pipe.layers])
    ev = np.stack([untile(lay.V, d, F, vbn).float().cpu().numpy() for lay in pipe.layers])
    ref, chosen = O.moe_forward(emb.cpu().numpy(), router, eu, ev)
    got = x.cpu().numpy()
    e0 = emb.cpu().numpy()
    err = float(np.abs(got - ref).max() / np.abs(ref).max())
    derr = float(np.abs((got - e0) - (ref - e0)).max() / np.abs(ref - e0).max())
    assert err < 1e-2 and derr < 1e-2, (err, derr)
    assert (pipe.route.cpu().numpy() == chosen).mean() >= 0.999


@pytest.mark.parametrize("replication,ffn,E,d,F", [("on", "auto", 32, 256, 512), ("off", "auto", 32, 256, 512),
                                                   ("on", "pair", 32, 256, 512), ("on", "two", 8, 768, 3072),
                                                   ("split", "pair", 8, 768, 3072)])
def test_step_graph_counts_its_kernels_and_replays_the_step(replication, ffn, E, d, F):
    """The captured step graph's kernel-node count (the launches bench.py reports) equals the
    engine's own host-side tally, and one replay gives the eager step's bits (d = 768 takes the
    fused rank + permute kernel)."""
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=3, num_experts=E, d_model=d, d_ff=F, tokens=4096, sru_layers=2,
                         capacity=64, replication=replication, ffn=ffn, seed=5)
    pipe = MoEPipeline(cfg)
    emb, _, _ = pipe.wl.batch(cfg.tokens)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        x_eager = emb.clone()
        pipe.step(x_eager)
        x = emb.clone()
        g = pipe.capture(x)
        x.copy_(emb)
        g.replay()
    torch.cuda.synchronize()
    assert g.launches == g.issued, (g.launches, g.issued)
    assert g.launches > 0
    assert torch.equal(x, x_eager)


def test_overlapped_pipeline_equals_sequential():
    """The two-stream schedule (predictor of batch i+1 on its own stream while batch i is planned,
    placed and forwarded; engine.OverlappedPipeline) gives the sequential schedule's bits: the
    analogue of the reference's mode_equivalence_check (src/pipeline.py:227-245) on the device path."""
    from paper_2605_11537_b200.engine import MoEPipeline, OverlappedPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=2,
                         capacity=64, predictor="random", seed=11)
    seq, ovl = MoEPipeline(cfg), MoEPipeline(cfg)
    batches = [seq.wl.batch(cfg.tokens)[0] for _ in range(4)]
    s = torch.cuda.Stream()
    outs, res = [], []
    with torch.cuda.stream(s):
        for b in batches:
            x = b.clone()
            seq.step(x)
            outs.append(x.clone())
            res.append(seq.res.clone())
    torch.cuda.synchronize()
    ov = OverlappedPipeline(ovl)
    ov.run(batches, 4)
    torch.cuda.synchronize()
    assert torch.equal(ov.xbuf[0], outs[2]) and torch.equal(ov.xbuf[1], outs[3])
    assert torch.equal(ovl.res, res[3])
    assert torch.equal(ov.assign[1], seq.assign)  # batch 3's predicted table


def test_fixed_split_expert_parallel_step_graph_and_rollback():
    """Fixed-split EP dispatch through a real NCCL group (world size 1, collectives forced):
    the eager step and a CUDA graph of the whole step (all-gathers and static all-to-alls
    captured) give the single-device step's bits; a split too small for the layers is
    detected once per step, rolled back (stream and residency) and re-run compactly."""
    import socket

    import torch.distributed as dist

    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                            device_id=torch.device("cuda", torch.cuda.current_device()))
    try:
        cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=3,
                             capacity=64, seed=5)
        a = MoEPipeline(cfg)
        emb, _, _ = a.wl.batch(cfg.tokens)
        xa = emb.clone()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            a.step(xa)
            b = MoEPipeline(cfg)
            b.enable_expert_parallel(peer_cap=None)
            b.force_collectives = True
            assert b.ep.k.peer_cap == cfg.tokens
            xb = emb.clone()
            b.step(xb)  # eager fixed-split step (plans residency for the replays below)
            torch.cuda.synchronize()
            assert torch.equal(xa, xb)
            g = b.capture(xb)
            for _ in range(2):
                xb.copy_(emb)
                g.replay()
            torch.cuda.synchronize()
            assert not b.ep_overflowed()
            assert torch.equal(xa, xb)
            g.destroy()  # a graph holding captured NCCL collectives goes before its process group
            # a fixed split of 64 rows cannot hold the layer: flagged, rolled back, re-run compactly
            c = MoEPipeline(cfg)
            c.enable_expert_parallel(peer_cap=64)
            c.force_collectives = True
            xc = emb.clone()
            c.step(xc)
            torch.cuda.synchronize()
            assert c.ep.k.peer_cap == 64 and not c.ep_overflowed()
            assert torch.equal(xa, xc)
            assert torch.equal(c.res, b.res)
    finally:
        dist.destroy_process_group()


def test_peer_memory_expert_parallel_step_graph_and_rollback():
    """Peer-memory EP (dispatch into the destination's receive block, combine fused into GEMM2's
    epilogue, device barriers) at world size 1 -- the peer tables hold this process's own buffers
    and the barrier waits only on itself: the eager step and a CUDA graph of the whole step give
    the single-device step's bits; an undersized split is rolled back and re-run compactly."""
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=3,
                         capacity=64, seed=5)
    a = MoEPipeline(cfg)
    emb, _, _ = a.wl.batch(cfg.tokens)
    xa = emb.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a.step(xa)
        b = MoEPipeline(cfg)
        b.enable_expert_parallel(peer_cap=None, p2p=True)
        assert b.ep.k.p2p and b.ep.k.peer_cap == cfg.tokens
        xb = emb.clone()
        b.step(xb)  # eager (maps the stream buffer; plans residency for the replays)
        torch.cuda.synchronize()
        assert torch.equal(xa, xb)
        g = b.capture(xb)
        for _ in range(2):
            xb.copy_(emb)
            g.replay()
        torch.cuda.synchronize()
        assert not b.ep_overflowed()
        assert torch.equal(xa, xb)
        assert int(b.ep.k.epoch.item()) == int(b.ep.k.flags[0].item()) > 0
        g.destroy()
        c = MoEPipeline(cfg)
        c.enable_expert_parallel(peer_cap=64, p2p=True)
        xc = emb.clone()
        c.step(xc)
        torch.cuda.synchronize()
        assert not c.ep_overflowed()
        assert torch.equal(xa, xc)


def test_peer_memory_setup_failure_falls_back_to_all_to_all(monkeypatch):
    """A peer mapping that cannot be made (or a failed start-up check) selects the all-to-all
    form of the same fixed-split layout -- and the step still gives the single-device bits."""
    from paper_2605_11537_b200 import ep as EP
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=2, num_experts=16, d_model=256, d_ff=512, tokens=2048, sru_layers=2,
                         capacity=32, seed=9)
    a = MoEPipeline(cfg)
    emb, _, _ = a.wl.batch(cfg.tokens)
    xa = emb.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        a.step(xa)
        for broken in ("connect", "verify_peers"):
            def fail(self, *args, **kwargs):
                raise RuntimeError("no peer access")
            with monkeypatch.context() as m:
                m.setattr(EP.CudaEpKernels, broken, fail)
                b = MoEPipeline(cfg)
                b.enable_expert_parallel(peer_cap=None, p2p=True)
            assert not b.ep_p2p and not b.ep.k.p2p and b.ep.k.peer_cap == cfg.tokens
            xb = emb.clone()
            b.step(xb)
            torch.cuda.synchronize()
            assert torch.equal(xa, xb)
