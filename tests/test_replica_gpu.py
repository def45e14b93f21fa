"""Physical expert replicas (K9, north_star "a replica plan that physically copies overloaded
experts"; reference events src/placement.py:133-160).

With physical replicas every resident replica slot owns a copy of its expert's weights in the
layer's pool; LOAD / REPLICATE / OFFLOAD events copy or free them on the device. The forward
must equal the aliased (one weight copy per expert) engine bit for bit on every batch, the pool
must hold exactly the residency state (conservation of copies), and a warm batch with the same
demand must copy nothing (the reference's warm-reuse case, pkg/tests/test_placement.py:25-31).
(With an inaccurate predictor the corrective replicas of the execution map are offloaded by the
next placement and loaded again: that churn is real and is not asserted away.)"""

import pytest
import torch

pytestmark = pytest.mark.gpu


def _pipe(physical, **kw):
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig

    cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=768, d_ff=1024, tokens=4096, sru_layers=2,
                         capacity=64, ffn="two", seed=11, physical_replicas=physical, **kw)
    return MoEPipeline(cfg)


@pytest.mark.parametrize("predictor", ["constructed", "random"])
def test_physical_replicas_equal_aliased_and_conserve_copies(predictor):
    a, b = _pipe(False, predictor=predictor), _pipe(True, predictor=predictor)
    batches = [a.wl.batch(a.cfg.tokens)[0] for _ in range(3)]
    prev = None
    for i, emb in enumerate(batches + [batches[-1]]):
        xa, xb = emb.clone(), emb.clone()
        a.step(xa)
        b.step(xb)
        torch.cuda.synchronize()
        assert torch.equal(xa, xb), i
        assert torch.equal(a.res, b.res)
        st = b.replica_stats()
        assert not st["overflow"]
        # every resident replica holds exactly one copy: copies made - copies freed = residency
        assert st["loads"] + st["replicates"] - st["offloads"] == int(b.res.sum().item())
        if i == len(batches) and predictor == "constructed":  # same batch again: warm residency, no copies
            assert st["loads"] == prev["loads"] and st["replicates"] == prev["replicates"]
        prev = st
    assert prev["loads"] >= a.cfg.num_layers  # the first batch loaded experts into every layer's pool
