"""Parity at the BASELINE shapes (VERDICT r01 "What's weak" 1): the production
kernels at d = 768, F = 3072 -- the 192-column GEMM2 with its 5-deep ring and reversed unit walk,
the CTA-pair kernels of config 2, the fused rank + permute kernel, the SRU scan at width 768 --
checked against the CPU oracle (oracle/moesim_oracle.py, pinned to the reference's golden
vectors), not against other variants of themselves.

MoE forward (reference router_oracle.py:119-135): every token's path through the layers is
independent of the other tokens (top-1 routing, ungated residual), so the oracle runs a seeded
sample of tokens of the full 16k-token batch the GPU processed (the GPU still builds every
replica, piece and tile of the whole batch). Tolerance: max-norm relative error <= 1e-2
(north star; bf16 operands, fp32 accumulation) on the output stream and on the layers' delta.

SRU (reference predictor.py:175-223): the scan is causal from c_0 = 0, so the first tokens of
the device's whole-batch scan are checked exactly against the float64 oracle on that prefix;
predicted-expert argmax flips are counted and bounded (the survey measured 2/512 at d = 768)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


class _DeviceExperts:
    """eu[l, e] / ev[l, e] for the oracle: one expert's weights untiled from the device layout
    (mp_tile_kmajor [E][N/bn][K/64][bn][64]) into float32 numpy on demand (bounded host RAM)."""

    def __init__(self, pipe, which):
        self.pipe, self.which, self.cache = pipe, which, {}

    def __getitem__(self, key):
        l, e = key
        if key not in self.cache:
            lay = self.pipe.layers[l]
            d, F = lay.dp, lay.Fp
            if self.which == "u":
                t, N, K, bn = lay.U, F, d, 256
            else:
                t, N, K, bn = lay.V, d, F, lay.vbn
            blk = t.view(lay.E, N // bn, K // 64, bn, 64)[e]
            self.cache[key] = blk.permute(0, 2, 1, 3).reshape(N, K).float().cpu().numpy()
        return self.cache[key]


def _flips_are_near_ties(got_assign, ref_assign, ref_h, heads, rel_gap=2e-2):
    """Predicted-expert argmax flips are counted, not failed (north star) -- but each one must be
    a near tie of the float64 logits: the expert the GPU chose scores within rel_gap x the row's
    largest |logit| of the oracle's choice (bf16 operands move logits by ~1e-3 relative)."""
    flips = np.argwhere(got_assign != ref_assign)
    for l, t in flips:
        z = ref_h[t] @ heads[l].T
        gap = z[ref_assign[l, t]] - z[got_assign[l, t]]
        assert gap <= rel_gap * np.abs(z).max(), (l, t, gap, np.abs(z).max())
    assert len(flips) <= 0.02 * ref_assign.size, len(flips)
    return len(flips)


def _pipeline(**kw):
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(**kw)
    return MoEPipeline(cfg)


def _check_moe(pipe, emb, x, sample, seed):
    from oracle import moesim_oracle as O

    rng = np.random.default_rng(seed)
    T, L = pipe.cfg.tokens, pipe.cfg.num_layers
    route = pipe.route.cpu().numpy()
    # the sample covers the hottest expert of every layer and a spread of cold ones
    hot = [int(np.flatnonzero(route[l] == np.bincount(route[l]).argmax())[0]) for l in range(L)]
    idx = np.unique(np.concatenate([rng.choice(T, size=sample, replace=False), hot]))
    router = np.stack([pipe.wl.router(l).cpu().numpy() for l in range(L)]).astype(np.float32)
    e0 = emb[idx].cpu().numpy()
    ref, chosen = O.moe_forward(e0, router, _DeviceExperts(pipe, "u"), _DeviceExperts(pipe, "v"))
    got = x[idx].cpu().numpy()
    assert (chosen == route[:, idx]).all(), "routing differs from the oracle's float64 argmax"
    err, derr = _rel(got, ref), _rel(got - e0, ref - e0)
    assert err <= TOL and derr <= TOL, (err, derr)
    return err, derr


def test_config3_shape_moe_forward_matches_oracle():
    """Switch-base-128 layer shape (E = 128, d = 768, F = 3072, 16,384 tokens, Zipf 1.2, C = 296,
    tile-unit demand), two MoE layers (host RAM), random predictor (corrective replicas), two
    batches (the second runs on the warm residency of the first)."""
    pipe = _pipeline(num_layers=2, num_experts=128, d_model=768, d_ff=3072, tokens=16384, sru_layers=2,
                     capacity=296, demand_unit=128, predictor="random", seed=21)
    assert pipe.cfg.ffn == "two"
    for k in range(2):
        emb, _, oracle_routes = pipe.wl.batch(pipe.cfg.tokens)
        x = emb.clone()
        pipe.step(x)
        torch.cuda.synchronize()
        assert torch.equal(pipe.route.long(), oracle_routes.long())
    _check_moe(pipe, emb, x, 384, seed=5)


@pytest.mark.parametrize("replication", ["on", "off"])
def test_config2_shape_cta_pair_moe_forward_matches_oracle(replication):
    """Switch-base-8 layer shape (E = 8, d = 768, F = 3072, 16,384 tokens: 2,048 per expert),
    where --ffn auto takes the CTA-pair (cta_group::2) grouped GEMMs."""
    pipe = _pipeline(num_layers=1, num_experts=8, d_model=768, d_ff=3072, tokens=16384, sru_layers=2,
                     capacity=148, demand_unit=128, replication=replication, seed=22)
    assert pipe.cfg.ffn == "pair"
    emb, _, _ = pipe.wl.batch(pipe.cfg.tokens)
    x = emb.clone()
    pipe.step(x)
    torch.cuda.synchronize()
    _check_moe(pipe, emb, x, 384, seed=6)


def test_engine_predictor_prefix_matches_fp64_oracle_at_d768():
    """The engine's predictor (10 SRU layers at d = 768 over a 16,384-token batch, heads for 12
    MoE layers x 128 experts): hidden states of the first 1,024 tokens vs the float64 oracle on
    that prefix (causal scan from c_0 = 0), and predicted-expert flips counted."""
    from oracle import moesim_oracle as O

    pipe = _pipeline(num_layers=12, num_experts=128, d_model=768, d_ff=256, tokens=16384, sru_layers=10,
                     capacity=296, predictor="random", seed=23)
    emb, _, _ = pipe.wl.batch(pipe.cfg.tokens)
    x = emb.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipe.predict(x, s.cuda_stream)
    torch.cuda.synchronize()
    P = 1024
    last = (pipe.cfg.sru_layers - 1) % 2
    got = pipe.h32[last][:P].double().cpu().numpy()
    ref_assign, ref_h = O.predict_assignment(emb[:P].double().cpu().numpy(), pipe.sru_host, pipe.heads_host)
    err = _rel(got, ref_h)
    assert err <= TOL, err
    _flips_are_near_ties(pipe.assign[:, :P].long().cpu().numpy(), ref_assign, ref_h, pipe.heads_host)
    assert int(pipe.nonfinite.item()) == 0


def test_public_sru_forward_and_predict_batch_at_d768():
    """The drop-in API (predictor.sru_forward / predict_batch) at d = 768, S = 10, T = 4,096,
    12 heads of 128 experts, vs the float64 oracle (reference predictor.py:175-223), on the
    reference workload's embeddings (workload.py:178-211: unit centroids + N(0, 0.1^2) noise,
    Zipf 1.2). Inputs of norm ~14 (standard normals x 0.5) reach 1.08e-2 here: bf16 operands
    scale the error with the pre-activation size."""
    from oracle import moesim_oracle as O
    from paper_2605_11537_b200.predictor import SruLayerParams, SruParams, predict_batch, sru_forward

    L, E, d, T, S = 12, 128, 768, 4096, 10
    layers, heads = O.init_sru_params(L, E, d, S, seed=31)
    params = SruParams([SruLayerParams(*lay) for lay in layers], heads)
    (x, _), = O.generate_trace(L, E, d, T, 1, 1.2, seed=32)
    ref_assign, ref_h = O.predict_assignment(x, layers, heads)
    h = sru_forward(x, params)
    err = _rel(h, ref_h)
    assert err <= TOL, err
    table = predict_batch(x, params)
    _flips_are_near_ties(table.assignment, ref_assign, ref_h, heads)
