"""Device-resident engine (MoEPipeline) on a small Switch-like workload: the layer-chained
router (GEMM2 epilogue writes the next layer's split operand and bound scale) must give
the same routing and residual stream, bit for bit, as the unchained pre-pass, and the
routing must be the workload's exact (reference float64) routing."""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(chain, ffn="two", replication="on"):
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=4, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=2,
                         capacity=64, chain_router=chain, ffn=ffn, replication=replication, seed=3)
    pipe = MoEPipeline(cfg)
    emb, _, oracle_routes = pipe.wl.batch(cfg.tokens)
    x = emb.clone()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        pipe.step(x)
    torch.cuda.synchronize()
    return x, pipe.route.clone(), oracle_routes


@pytest.mark.parametrize("replication", ["on", "off"])
def test_chained_router_is_bitwise_identical(replication):
    x1, r1, oracle = _run(True, replication=replication)
    x0, r0, _ = _run(False, replication=replication)
    assert torch.equal(r1, r0)
    assert (r1.long() == oracle.long()).all()
    assert torch.equal(x1, x0)
