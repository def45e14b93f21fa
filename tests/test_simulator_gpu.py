"""Cost-model metrics from device counts: the drop-in BatchRunner /
simulate_strategy (paper_2605_11537_b200/simulator.py, counts by csrc/counts.cu) against
the reference's own Metrics (tests/golden/metrics.json, written by the reference's
simulate_strategy, src/simulator.py:210-273), and the engine's per-step counts against a
host recount of the same device arrays."""

import json
from dataclasses import asdict
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import moesim_oracle as O

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _trace(case):
    from paper_2605_11537_b200.workload import Batch, ModelShape, RoutingTrace

    L, E, d, T = case["L"], case["E"], case["d"], case["T"]
    gen = case["gen"]
    if gen["kind"] == "hot":
        pairs = O.generate_hot_trace(L, E, d, T, 4, gen["num_hot"], case["seed"])
    else:
        pairs = O.generate_trace(L, E, d, T, 4, gen["skew"], case["seed"])
    batches = [Batch(i, e, np.asarray(r, dtype=np.int64)) for i, (e, r) in enumerate(pairs)]
    return RoutingTrace(ModelShape(L, E, d, T), batches)


def _close(a: dict, b: dict, exact: bool):
    for k, v in b.items():
        if exact:
            assert a[k] == v, (k, a[k], v)
        else:
            assert a[k] == pytest.approx(v, rel=1e-12, abs=1e-12), (k, a[k], v)


def test_batch_runner_metrics_match_reference():
    from paper_2605_11537_b200.predictor import HashTable, init_params
    from paper_2605_11537_b200.simulator import BatchRunner, CostModel, aggregate_metrics

    cases = json.loads((G / "metrics.json").read_text())
    assert len(cases) == 60
    for case in cases:
        trace = _trace(case)
        params = init_params(case["L"], case["E"], case["d"], num_sru_layers=2, seed=case["seed"]) \
            if case["sru"] else "oracle"
        cost = CostModel(*case["cost"])
        exact = all(float(c).is_integer() for c in case["cost"])
        runner = BatchRunner(trace, case["strategy"], case["capacity"], params=params, cost=cost)
        per_batch = []
        for batch, ref in zip(trace.batches, case["batches"]):
            # the reference's (fp64) predicted table; the GPU predictor is checked in test_parity_gpu
            table = HashTable.from_assignment(batch.index, np.array(ref["table"], dtype=np.int64))
            m = runner.run_batch(batch, table).metrics
            _close(asdict(m), ref["metrics"], exact)
            per_batch.append(m)
        _close(asdict(aggregate_metrics(per_batch)), case["aggregate"], exact)


def test_simulate_layer_known_answers():
    from paper_2605_11537_b200.errors import ConfigurationError
    from paper_2605_11537_b200.placement import TransferEvent
    from paper_2605_11537_b200.simulator import CostModel, simulate_layer

    assert simulate_layer(np.repeat([0, 1], 32), 2, [], CostModel()) == (32.0, 64.0)
    assert simulate_layer(np.arange(7), 7, [], CostModel()) == (1.0, 7.0)
    ev = [TransferEvent("load", 0, 1, 0), TransferEvent("replicate", 0, 1, 1), TransferEvent("offload", 0, 2, 0)]
    assert simulate_layer(np.array([0, 0, 1]), 2, ev, CostModel()) == (10.0 + 2.0 + 5.0 + 2.0, 3.0)
    with pytest.raises(ConfigurationError):
        simulate_layer(np.array([], dtype=np.int64), 1, [], CostModel())
    with pytest.raises(ConfigurationError):
        simulate_layer(np.array([0, 3]), 3 - 1, [], CostModel())


def test_engine_counts_and_metrics():
    """MoEPipeline.metrics: device counts of a real step equal a host recount of the engine's own
    device arrays, and the Metrics follow the reference formulas from those counts."""
    from paper_2605_11537_b200 import _lib
    from paper_2605_11537_b200.engine import MoEPipeline, PipelineConfig
    from paper_2605_11537_b200.simulator import CostModel

    cfg = PipelineConfig(num_layers=3, num_experts=32, d_model=256, d_ff=512, tokens=4096, sru_layers=2,
                         capacity=64, predictor="random", seed=5)
    pipe = MoEPipeline(cfg)
    s = torch.cuda.Stream()
    cost = CostModel(1.0, 10.0, 2.0, 5.0)
    with torch.cuda.stream(s):
        pipe.step(pipe.wl.batch(cfg.tokens)[0])
        torch.cuda.synchronize()
        _, cold = pipe.metrics(cost)
        assert (cold[:, 0] > 0).all()  # cold start: every layer loads its experts
        pipe.step(pipe.wl.batch(cfg.tokens)[0])  # warm residency
        torch.cuda.synchronize()
        m, counts = pipe.metrics(cost)
    ev = pipe.pred_event.cpu().numpy()
    kind = np.where(ev >= 0, ev >> _lib.MP_EVENT_KIND_SHIFT, 0)
    tts = pipe.exec_slot.cpu().numpy()
    ns = pipe.exec_slots.cpu().numpy()
    T = cfg.tokens
    lat = slot_time = transfer_total = 0.0
    mks = []
    for l in range(cfg.num_layers):
        loads = int((kind[l] == _lib.MP_EVENT_LOAD).sum() + pipe.corrective[l].sum().item())
        reps = int((kind[l] == _lib.MP_EVENT_REPLICATE).sum())
        offl = int(pipe.offloads[l].sum().item())
        q = np.bincount(tts[l], minlength=int(ns[l]))
        assert len(q) == ns[l]
        assert counts[l].tolist() == [loads, reps, offl, int(q.max()), int(ns[l])]
        transfer = 10.0 * loads + 2.0 * reps + 5.0 * offl
        mk = transfer + float(q.max())
        mks.append(mk)
        lat += mk
        slot_time += ns[l] * mk
        transfer_total += transfer
    assert m.batch_latency == lat and m.transfer_time == transfer_total and m.slot_time == slot_time
    assert m.busy_time == float(cfg.num_layers * T) and m.num_tokens == T
    assert m.utilization == min(1.0, m.busy_time / slot_time)
    acc = float((pipe.assign == pipe.route).float().mean().item())
    assert m.prediction_accuracy == acc < 1.0  # random predictor
    # measured layer times replace the cost-model makespans
    mm, _ = pipe.metrics(cost, layer_latency=[0.25] * cfg.num_layers)
    assert mm.batch_latency == 0.75 and mm.throughput == T / 0.75
    # each layer's cost-model times rescaled to its given makespan: per-layer utilization kept
    busy_ms = sum(T * 0.25 / mk for mk in mks)
    assert mm.busy_time == pytest.approx(busy_ms, rel=1e-12)
    assert mm.utilization == pytest.approx(min(1.0, busy_ms / sum(0.25 * n for n in ns)), rel=1e-12)
