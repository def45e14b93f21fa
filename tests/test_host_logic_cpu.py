"""Host-side logic of the simulator / pipeline drop-ins (no GPU): the queue schedule of the
two-actor pipeline (reference src/pipeline.py:70-90, known answers of pkg/tests/test_pipeline.py)
and the reference cost model evaluated on per-layer counts (src/simulator.py:62-81, 210-235)."""

import numpy as np
import pytest

from paper_2605_11537_b200.errors import ConfigurationError, MetricError
from paper_2605_11537_b200.pipeline import PipelineConfig, compute_schedule
from paper_2605_11537_b200.simulator import CostModel, aggregate_metrics, metrics_from_counts, utilization


def test_schedule_known_answers():
    dq, stalls, total = compute_schedule(2.0, [5.0, 5.0, 5.0], 1)
    assert (dq, stalls, total) == ([2.0, 7.0, 12.0], [2.0, 0.0, 0.0], 17.0)
    _, stalls, total = compute_schedule(8.0, [5.0, 5.0, 5.0], 2)
    assert (stalls, total) == ([8.0, 3.0, 3.0], 29.0)
    _, stalls, total = compute_schedule(0.0, [5.0, 4.0, 3.0], 10)
    assert (stalls, total) == ([0.0, 0.0, 0.0], 12.0)
    with pytest.raises(ConfigurationError):
        compute_schedule(1.0, [1.0], 0)


def test_schedule_bounds(rng):
    for _ in range(300):
        n = int(rng.integers(1, 12))
        build = float(rng.uniform(0, 5))
        inf = [float(rng.uniform(0.5, 5)) for _ in range(n)]
        cap = int(rng.integers(1, 4))
        dq, stalls, total = compute_schedule(build, inf, cap)
        assert total >= max(sum(inf), n * build) - 1e-9
        assert total == pytest.approx(sum(inf) + sum(stalls))
        assert all(s >= 0 for s in stalls) and dq == sorted(dq)


def test_pipeline_config_validation():
    with pytest.raises(ConfigurationError):
        PipelineConfig(queue_capacity=0)
    with pytest.raises(ConfigurationError):
        PipelineConfig(mode="threads")
    with pytest.raises(ConfigurationError):
        PipelineConfig(hash_build_cost=-1.0)


def test_metrics_from_counts_follow_the_reference_formulas():
    # two layers: {loads, replicates, offloads, longest queue, slots}
    counts = np.array([[2, 1, 3, 40, 9], [0, 4, 0, 25, 12]])
    cost = CostModel(t_compute=1.0, t_load=10.0, t_replicate=2.0, t_offload=5.0)
    m = metrics_from_counts(counts, 100, cost, 0.75)
    mk0, mk1 = 2 * 10 + 2 + 3 * 5 + 40.0, 4 * 2 + 25.0
    assert m.batch_latency == mk0 + mk1
    assert m.transfer_time == (2 * 10 + 2 + 15) + 8
    assert m.busy_time == 200.0 and m.num_tokens == 100
    assert m.slot_time == 9 * mk0 + 12 * mk1
    assert m.utilization == min(1.0, 200.0 / m.slot_time)
    assert m.throughput == 100 / m.batch_latency and m.prediction_accuracy == 0.75
    # measured layer times: the layer's cost-model times rescale, its utilization is kept
    mm = metrics_from_counts(counts, 100, cost, 0.75, layer_latency=[2.0, 1.0])
    assert mm.batch_latency == 3.0
    assert mm.busy_time == pytest.approx(100 * 2.0 / mk0 + 100 * 1.0 / mk1)
    assert aggregate_metrics([m, m]).batch_latency == 2 * m.batch_latency


def test_cost_model_errors():
    with pytest.raises(ConfigurationError):
        CostModel(t_load=-1.0)
    with pytest.raises(MetricError):
        utilization(1.0, 1, 0.0)
    with pytest.raises(MetricError):
        metrics_from_counts(np.zeros((1, 5), dtype=np.int64), 4, CostModel(t_compute=0.0), 1.0)
    with pytest.raises(MetricError):
        aggregate_metrics([])
