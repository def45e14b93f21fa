"""Cost-model metrics from DEVICE counts: drop-in for the reference's BatchRunner /
simulate_strategy (src/simulator.py:36-273), SURVEY.md §8(f) rank 2.

The reference charges every layer ``transfer + longest_queue * t_compute`` where
``transfer`` sums the layer's LOAD / REPLICATE / OFFLOAD events (src/simulator.py:62-81)
and the longest queue is the busiest replica slot of the execution map. Here the
planner, the placement walk and the execution map run on the GPU (planner.py,
placement.py) and one kernel (``mp_layer_counts``, csrc/counts.cu) reduces their
device outputs -- per-token event codes, per-expert offloads and corrective loads,
the token -> slot map -- to five counts per layer. The host only turns those counts
into the reference's ``Metrics`` (``metrics_from_counts``).

Arithmetic: the reference adds event costs one by one in log order; here a layer's
transfer time is ``n_load * t_load + n_replicate * t_replicate + n_offload * t_offload``
(exactly rounded with ``math.fsum``). The two are equal bit for bit whenever the costs
are integers (the reference default ``CostModel()``); otherwise they agree to within one
rounding per event.

``MoEPipeline.metrics`` (engine.py) feeds the same counts from the benchmarked step, and
can swap the cost-model layer time for the measured one.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import ptr, require_device, stream_ptr
from .errors import ConfigurationError, MetricError
from .placement import LOAD, OFFLOAD, REPLICATE, DeviceState, TransferLog, apply_batch, execution_map
from .planner import ReplicaPlan, check_positive, plan_layers_with_fallback
from .predictor import HashTable, SruParams, evaluate_accuracy, predict_batch
from .router_oracle import LayerPlacement, Placement

RESIDENT_ALL = "resident-all"
DISTINCT_ONLY = "distinct-only"
REPLICATED = "replicated"
STRATEGIES = (RESIDENT_ALL, DISTINCT_ONLY, REPLICATED)

ORACLE_PREDICTOR = "oracle"

# columns of mp_layer_counts
C_LOADS, C_REPLICATES, C_OFFLOADS, C_QUEUE, C_SLOTS = range(5)


def check_nonnegative(name: str, value: float) -> float:
    """src/validation.py:15-19."""
    value = float(value)
    if value < 0:
        raise ConfigurationError(f"{name} must be >= 0, got {value}")
    return value


@dataclass(frozen=True)
class CostModel:
    """Abstract time units of the simulated device (src/simulator.py:36-49)."""

    t_compute: float = 1.0
    t_load: float = 10.0
    t_replicate: float = 2.0
    t_offload: float = 5.0

    def __post_init__(self):
        for name in ("t_compute", "t_load", "t_replicate", "t_offload"):
            check_nonnegative(name, getattr(self, name))

    def event_cost(self, kind: str) -> float:
        return {LOAD: self.t_load, REPLICATE: self.t_replicate, OFFLOAD: self.t_offload}[kind]

    def transfer_time(self, loads: int, replicates: int, offloads: int) -> float:
        """Cost of a layer's events from their counts (see the module note on rounding)."""
        return math.fsum((loads * self.t_load, replicates * self.t_replicate, offloads * self.t_offload))


@dataclass
class Metrics:
    """src/simulator.py:52-62 (same fields, same meaning)."""

    batch_latency: float
    throughput: float
    utilization: float
    stall_time: float
    transfer_time: float
    busy_time: float
    slot_time: float
    num_tokens: int
    prediction_accuracy: float


def layer_counts(token_to_slot: torch.Tensor, num_slots: torch.Tensor, max_slots: int,
                 token_event: torch.Tensor | None = None, offloads: torch.Tensor | None = None,
                 corrective: torch.Tensor | None = None) -> np.ndarray:
    """(L, 5) int64 counts {loads, replicates, offloads, longest queue, slots} of device arrays
    (token_to_slot / token_event: L x T, offloads / corrective: L x E, num_slots: L)."""
    dev = token_to_slot.device
    token_to_slot, num_slots = token_to_slot.contiguous(), num_slots.contiguous()
    token_event = token_event.contiguous() if token_event is not None else None
    offloads = offloads.contiguous() if offloads is not None else None
    corrective = corrective.contiguous() if corrective is not None else None
    L, T = token_to_slot.shape
    counts = torch.empty(L, 5, dtype=torch.int32, device=dev)
    err = torch.zeros(1, dtype=torch.int32, device=dev)
    e_off = offloads.shape[1] if offloads is not None else 0
    e_corr = corrective.shape[1] if corrective is not None else 0
    _lib.call("mp_layer_counts", ptr(token_event) if token_event is not None else None,
              ptr(offloads) if offloads is not None else None, ptr(corrective) if corrective is not None else None,
              ptr(token_to_slot), ptr(num_slots), L, T, e_off, e_corr, int(max_slots), ptr(counts), ptr(err),
              stream_ptr())
    out = counts.cpu().numpy().astype(np.int64)
    if int(err.item()):
        raise ConfigurationError("token map refers to slots outside [0, num_slots)")
    return out


def layer_times(counts: np.ndarray, num_tokens: int, cost: CostModel) -> list[tuple[float, float, float, int]]:
    """Per layer (makespan, transfer, busy, slots) of the reference cost model
    (simulate_layer, src/simulator.py:62-81)."""
    rows = []
    for c in counts:
        transfer = cost.transfer_time(int(c[C_LOADS]), int(c[C_REPLICATES]), int(c[C_OFFLOADS]))
        makespan = transfer + float(c[C_QUEUE]) * cost.t_compute
        rows.append((makespan, transfer, float(num_tokens) * cost.t_compute, int(c[C_SLOTS])))
    return rows


def metrics_from_counts(counts: np.ndarray, num_tokens: int, cost: CostModel, accuracy: float,
                        layer_latency: list[float] | None = None) -> Metrics:
    """BatchRunner._metrics_from (src/simulator.py:210-235) over device counts. With
    ``layer_latency`` (e.g. measured ms per MoE layer) each layer's cost-model times are rescaled
    so that its makespan is the given time (transfer and busy time in the same unit; the layer's
    utilization is unchanged)."""
    latency = transfer_total = busy_total = slot_time = 0.0
    for l, (makespan, transfer, busy, slots) in enumerate(layer_times(counts, num_tokens, cost)):
        if layer_latency is not None:
            scale = float(layer_latency[l]) / makespan if makespan > 0 else 0.0
            makespan, transfer, busy = float(layer_latency[l]), transfer * scale, busy * scale
        latency += makespan
        transfer_total += transfer
        busy_total += busy
        slot_time += slots * makespan
    if latency <= 0 or slot_time <= 0:
        raise MetricError("batch latency is zero; set a positive t_compute")
    return Metrics(
        batch_latency=latency,
        throughput=num_tokens / latency,
        utilization=min(1.0, busy_total / slot_time),
        stall_time=0.0,
        transfer_time=transfer_total,
        busy_time=busy_total,
        slot_time=slot_time,
        num_tokens=num_tokens,
        prediction_accuracy=accuracy,
    )


def simulate_layer(token_to_slot, num_slots: int, events, cost: CostModel):
    """(makespan, busy_time) of one layer (src/simulator.py:62-81): the longest slot queue is
    counted on the device."""
    tts = np.asarray(token_to_slot, dtype=np.int64)
    if tts.size == 0:
        raise ConfigurationError("token map must be nonempty")
    if num_slots < 1 or tts.max() >= num_slots or tts.min() < 0:
        raise ConfigurationError("token map refers to slots outside [0, num_slots)")
    dev = require_device()
    d_tts = torch.from_numpy(np.ascontiguousarray(tts, dtype=np.int32).reshape(1, -1)).to(dev)
    d_ns = torch.full((1,), int(num_slots), dtype=torch.int32, device=dev)
    c = layer_counts(d_tts, d_ns, int(num_slots))
    transfer = sum(cost.event_cost(e.kind) for e in events)
    makespan = transfer + float(c[0, C_QUEUE]) * cost.t_compute
    busy = float(tts.size) * cost.t_compute
    return makespan, busy


def utilization(busy_time: float, num_slots: int, makespan: float) -> float:
    """busy / (slots * makespan), clamped to [0, 1] (src/simulator.py:84-89)."""
    if makespan <= 0:
        raise MetricError("utilization is undefined for zero makespan")
    check_positive("num_slots", num_slots)
    return float(min(1.0, max(0.0, busy_time / (num_slots * makespan))))


def normalize_strategy(name: str) -> str:
    if name == "distinct":
        return DISTINCT_ONLY
    if name not in STRATEGIES:
        raise ConfigurationError(f"unknown strategy {name!r}; expected one of {STRATEGIES}")
    return name


@dataclass
class BatchOutcome:
    """Everything one batch produced (src/simulator.py:100-107)."""

    table: HashTable
    placement: Placement
    log: TransferLog
    metrics: Metrics


class BatchRunner:
    """Stateful executor of one strategy over consecutive batches (src/simulator.py:110-208).

    Prediction (SRU), planning, placement and the execution map run on the GPU through this
    package's drop-in functions; the metrics come from ``mp_layer_counts`` over their device
    outputs."""

    def __init__(self, trace, strategy: str, capacity: int, params=ORACLE_PREDICTOR, cost: CostModel | None = None):
        self.strategy = normalize_strategy(strategy)
        self.trace = trace
        self.params = params
        self.cost = cost if cost is not None else CostModel()
        experts = trace.shape.experts_per_layer
        if self.strategy == RESIDENT_ALL:
            self.capacity = experts  # baseline keeps the whole layer resident
        else:
            self.capacity = check_positive("capacity", capacity)
        self.state = DeviceState(trace.shape.num_layers, self.capacity)
        self._warm = False

    def build_table(self, batch) -> HashTable:
        if isinstance(self.params, SruParams):
            return predict_batch(batch, self.params)
        if isinstance(self.params, str) and self.params == ORACLE_PREDICTOR:
            return HashTable.from_assignment(batch.index, batch.oracle_routing)
        raise ConfigurationError("params must be SruParams or 'oracle'")

    def _plan(self, table: HashTable) -> ReplicaPlan:
        """BatchRunner._plan (src/simulator.py:135-146) on the GPU planner: distinct-only caps, or
        capped replicas with an empty (fallback) plan for an infeasible layer."""
        return plan_layers_with_fallback(table, self.capacity, distinct_only=self.strategy == DISTINCT_ONLY)

    def run_batch(self, batch, table: HashTable | None = None) -> BatchOutcome:
        if table is None:
            table = self.build_table(batch)
        if self.strategy == RESIDENT_ALL:
            return self._run_resident_all(batch, table)
        return self._run_predicted(batch, table)

    def _accuracy_of(self, table: HashTable, batch) -> float:
        if isinstance(self.params, SruParams):
            return evaluate_accuracy(table.assignment, batch.oracle_routing)
        return 1.0

    def _run_resident_all(self, batch, table: HashTable) -> BatchOutcome:
        shape = self.trace.shape
        L, E = shape.num_layers, shape.experts_per_layer
        log = TransferLog()
        warm = not self._warm
        if warm:
            for layer in range(L):
                for expert in range(E):
                    self.state.add_replica(layer, expert)
                    log.record(LOAD, layer, expert, 0)
            self._warm = True
        routing = np.asarray(batch.oracle_routing, dtype=np.int64)
        layers = [LayerPlacement(slots=self.state.slots(l), token_to_slot=routing[l]) for l in range(L)]
        dev = require_device()
        d_tts = torch.from_numpy(np.ascontiguousarray(routing, dtype=np.int32)).to(dev)
        d_ns = torch.full((L,), E, dtype=torch.int32, device=dev)
        warm_loads = torch.ones(L, E, dtype=torch.int32, device=dev) if warm else None
        counts = layer_counts(d_tts, d_ns, E, corrective=warm_loads)
        metrics = metrics_from_counts(counts, shape.batch_size, self.cost, self._accuracy_of(table, batch))
        return BatchOutcome(table, Placement(layers=layers), log, metrics)

    def _run_predicted(self, batch, table: HashTable) -> BatchOutcome:
        plan = self._plan(table)
        self.state.last_place_device = self.state.last_exec_device = None
        _, placement, log = apply_batch(self.state, table, plan)
        place = self.state.last_place_device
        # tokens execute on their true experts; a miss loads the expert first (corrective LOAD)
        _, execution, xlog = execution_map(self.state, batch.oracle_routing)
        log.extend(xlog)
        ex = self.state.last_exec_device
        if ex is None:  # no tokens: simulate_layer rejects an empty token map (src/simulator.py:70-71)
            raise ConfigurationError("token map must be nonempty")
        full = place is not None and place["layers"] == list(range(table.num_layers))
        counts = layer_counts(ex["token_to_slot"], ex["num_slots"], ex["max_slots"],
                              token_event=place["token_event"][:, :ex["T"]] if full else None,
                              offloads=place["offloads"] if full else None, corrective=ex["corrective"])
        metrics = metrics_from_counts(counts, self.trace.shape.batch_size, self.cost,
                                      self._accuracy_of(table, batch))
        return BatchOutcome(table, placement, log, metrics)


@dataclass
class StrategyResult:
    strategy: str
    per_batch: list[Metrics]
    aggregate: Metrics


def aggregate_metrics(per_batch: list[Metrics]) -> Metrics:
    """Totals over batches; utilization time-weighted by slot time, stalls added to the latency
    (src/simulator.py:245-265)."""
    if not per_batch:
        raise MetricError("cannot aggregate zero batches")
    tot = {f: sum(getattr(m, f) for m in per_batch)
           for f in ("batch_latency", "stall_time", "transfer_time", "busy_time", "slot_time", "num_tokens")}
    latency = sum(m.batch_latency + m.stall_time for m in per_batch)  # per-batch sums, in batch order
    if latency <= 0 or tot["slot_time"] <= 0:
        raise MetricError("aggregate latency must be positive")
    return Metrics(batch_latency=latency, throughput=tot["num_tokens"] / latency,
                   utilization=min(1.0, tot["busy_time"] / tot["slot_time"]), stall_time=tot["stall_time"],
                   transfer_time=tot["transfer_time"], busy_time=tot["busy_time"], slot_time=tot["slot_time"],
                   num_tokens=tot["num_tokens"],
                   prediction_accuracy=float(np.mean([m.prediction_accuracy for m in per_batch])))


def simulate_strategy(trace, strategy: str, capacity: int, params=ORACLE_PREDICTOR,
                      cost: CostModel | None = None) -> StrategyResult:
    """Every batch of a trace under one residency strategy (src/simulator.py:268-273)."""
    runner = BatchRunner(trace, strategy, capacity, params, cost)
    per_batch = [runner.run_batch(batch).metrics for batch in trace.batches]
    return StrategyResult(runner.strategy, per_batch, aggregate_metrics(per_batch))


METRICS_COLUMNS = ["batch", "strategy", "experts", "capacity", "num_tokens", "latency", "throughput", "utilization",
                   "stall", "transfer_time", "prediction_accuracy", "busy_time", "slot_time"]


def metrics_row(batch: int, strategy: str, experts: int, capacity: int, m: Metrics) -> dict:
    """One row of the reference's metrics CSV (src/report.py:11-25, 47-62), the input of its
    ``summarize`` (src/report.py:100-148)."""
    return {"batch": batch, "strategy": strategy, "experts": experts, "capacity": capacity,
            "num_tokens": m.num_tokens, "latency": m.batch_latency, "throughput": m.throughput,
            "utilization": m.utilization, "stall": m.stall_time, "transfer_time": m.transfer_time,
            "prediction_accuracy": m.prediction_accuracy, "busy_time": m.busy_time, "slot_time": m.slot_time}
