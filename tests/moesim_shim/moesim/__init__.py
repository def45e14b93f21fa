"""Test-only import shim: ``import moesim`` resolves to this repository's drop-in API, so the
reference's own test files run unmodified against the GPU path (tools/run_reference_tests.sh).

Hot-path names come from ``paper_2605_11537_b200``. The synthetic trace generators are not part
of the hot path; for the tests they are the CPU oracle's restatements of
src/workload.py:228-313 (oracle/moesim_oracle.py), wrapped into this repository's
``RoutingTrace`` / ``Batch`` types."""

import numpy as np

from oracle import moesim_oracle as _O
from paper_2605_11537_b200.errors import (  # noqa: F401
    AggregationError,
    ConfigurationError,
    DeviceError,
    InfeasibleCapacityError,
    MetricError,
    MoesimError,
    NumericError,
    PlacementError,
    TraceParseError,
    TrainingError,
    ValidationError,
)
from paper_2605_11537_b200.placement import DeviceState, TransferEvent, TransferLog, apply_batch, apply_layer  # noqa: F401
from paper_2605_11537_b200.planner import ReplicaPlan, cap_replicas, demand_counts, plan_all_layers  # noqa: F401
from paper_2605_11537_b200.predictor import (  # noqa: F401
    HashTable,
    SruLayerParams,
    SruParams,
    SruState,
    evaluate_accuracy,
    init_params,
    predict_batch,
    sparsemax,
    sru_cell,
    sru_forward,
)
from paper_2605_11537_b200.router_oracle import (  # noqa: F401
    LayerPlacement,
    Placement,
    ToyMoeParams,
    expert_forward,
    moe_forward,
    oracle_route_batch,
    route_top1,
)
from paper_2605_11537_b200.pipeline import PipelineConfig, mode_equivalence_check, run_pipeline  # noqa: F401
from paper_2605_11537_b200.simulator import (  # noqa: F401
    BatchRunner,
    CostModel,
    Metrics,
    simulate_layer,
    simulate_strategy,
    utilization,
)
from paper_2605_11537_b200.training import TrainingResult, train_predictor  # noqa: F401
from paper_2605_11537_b200.workload import Batch, ModelShape, RoutingTrace  # noqa: F401


def _trace(shape, pairs, skew=0.0, seed=0, hot=0):
    batches = [Batch(i, emb, np.asarray(route, dtype=np.int64)) for i, (emb, route) in enumerate(pairs)]
    return RoutingTrace(shape, batches, skew=float(skew), seed=int(seed), hot_experts=int(hot))


def generate_trace(shape, num_batches, skew, seed, noise_scale=0.1):
    if num_batches < 1:
        raise ConfigurationError(f"num_batches must be >= 1, got {num_batches}")
    if skew < 0:
        raise ConfigurationError(f"skew must be >= 0, got {skew}")
    pairs = _O.generate_trace(shape.num_layers, shape.experts_per_layer, shape.d_model, shape.batch_size,
                              num_batches, skew, seed, noise_scale)
    return _trace(shape, pairs, skew, seed)


def generate_hot_trace(shape, num_batches, num_hot, seed, noise_scale=0.1):
    if num_batches < 1 or num_hot < 1:
        raise ConfigurationError("num_batches and num_hot must be >= 1")
    if num_hot > shape.experts_per_layer:
        raise ConfigurationError("num_hot cannot exceed experts_per_layer")
    pairs = _O.generate_hot_trace(shape.num_layers, shape.experts_per_layer, shape.d_model, shape.batch_size,
                                  num_batches, num_hot, seed, noise_scale)
    return _trace(shape, pairs, 0.0, seed, num_hot)


def oracle_params_for_trace(trace, d_ff=None):
    s = trace.shape
    r, u, v = _O.oracle_params_for_trace(s.num_layers, s.experts_per_layer, s.d_model, trace.seed, d_ff=d_ff)
    return ToyMoeParams(r, u, v)
