"""Capacity capping -- drop-in for ``moesim.planner`` (reference src/planner.py:1-85).

``cap_replicas`` / ``plan_all_layers`` run the on-device water-fill
(mp_cap_replicas), which is bit-exact with the reference's greedy grant loop
(src/planner.py:63-72; closed form SURVEY.md F4). Histograms come from
mp_histogram. Exceptions, layer tags and dict outputs match the reference.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import ptr, require_device, stream_ptr
from .errors import ConfigurationError, InfeasibleCapacityError
from .predictor import HashTable, _histograms, device_histograms


def check_positive(name: str, value, minimum: int = 1) -> int:
    """src/validation.py:8-12."""
    value = int(value)
    if value < minimum:
        raise ConfigurationError(f"{name} must be >= {minimum}, got {value}")
    return value


@dataclass
class ReplicaPlan:
    """Capped replica counts per (layer, expert); sum per layer <= capacity (src/planner.py:19-24)."""

    capacity: int
    layers: list[dict[int, int]]


def demand_counts(table: HashTable, layer: int) -> dict[int, int]:
    """Histogram of the table's layer row: expert -> number of assigned tokens (src/planner.py:27-33)."""
    if layer < 0 or layer >= table.num_layers:
        raise ConfigurationError(f"layer {layer} outside [0, {table.num_layers})")
    return _histograms(np.asarray(table.assignment[layer: layer + 1]))[0]


def cap_device(demand: torch.Tensor, capacity: int, unit_rows: int = 1):
    """(L, E) int32 device demand -> ((L, E) caps, (L,) infeasible flags), on device."""
    L, E = demand.shape
    caps = torch.empty_like(demand)
    inf = torch.empty(L, dtype=torch.int32, device=demand.device)
    _lib.call("mp_cap_replicas", ptr(demand), L, E, int(capacity), int(unit_rows), ptr(caps), ptr(inf),
              stream_ptr())
    return caps, inf


def cap_replicas(demand: dict[int, int], capacity: int) -> dict[int, int]:
    """Cap one layer's demand to ``capacity`` total replicas (src/planner.py:36-72).

    Raises InfeasibleCapacityError when even one replica per distinct expert
    does not fit; the placement layer owns the distinct-only fallback.
    """
    check_positive("capacity", capacity)
    experts = sorted(demand)
    if not experts:
        return {}
    if any(demand[e] < 1 for e in experts):
        raise InfeasibleCapacityError("demand counts must be >= 1")
    dev = require_device()
    # experts are compressed to their sorted order: the water-fill only uses id order
    d = torch.tensor([[int(demand[e]) for e in experts]], dtype=torch.int32, device=dev)
    caps, inf = cap_device(d, capacity)
    if int(inf.item()):
        raise InfeasibleCapacityError(f"{len(experts)} distinct experts exceed capacity {capacity}")
    return {e: int(c) for e, c in zip(experts, caps[0].cpu().tolist())}


def plan_all_layers(table: HashTable, capacity: int) -> ReplicaPlan:
    """Apply cap_replicas to every layer; errors identify the failing layer (src/planner.py:75-85)."""
    check_positive("capacity", capacity)
    L = table.num_layers
    if table.num_tokens == 0:
        return ReplicaPlan(capacity=capacity, layers=[{} for _ in range(L)])
    a = table.assignment
    E = int(a.max()) + 1
    if E > 1 << 16:
        ids, inv = np.unique(a, return_inverse=True)
        dev_a = torch.from_numpy(inv.reshape(a.shape).astype(np.int32)).to(require_device())
        E = len(ids)
    else:
        ids = None
        dev_a = table.device_assignment()
    demand = device_histograms(dev_a, E)
    caps, inf = cap_device(demand, capacity)
    inf = inf.cpu().numpy()
    bad = np.nonzero(inf)[0]
    if bad.size:
        l = int(bad[0])
        distinct = int((demand[l] > 0).sum().item())
        raise InfeasibleCapacityError(f"{distinct} distinct experts exceed capacity {capacity}", layer=l)
    caps = caps.cpu().numpy()
    layers = []
    for row in caps:
        nz = np.nonzero(row)[0]
        keys = nz if ids is None else ids[nz]
        layers.append({int(e): int(c) for e, c in zip(keys, row[nz])})
    return ReplicaPlan(capacity=capacity, layers=layers)


def plan_layers_with_fallback(table: HashTable, capacity: int, distinct_only: bool = False) -> ReplicaPlan:
    """BatchRunner._plan (src/simulator.py:135-146): per-layer caps; an infeasible layer gets
    an empty plan (apply_layer then falls back to distinct-only and flags it);
    ``distinct_only`` gives every demanded expert exactly one replica."""
    check_positive("capacity", capacity)
    L = table.num_layers
    if table.num_tokens == 0:
        return ReplicaPlan(capacity=capacity, layers=[{} for _ in range(L)])
    a = table.assignment
    E = int(a.max()) + 1
    if E > 1 << 16:
        ids, inv = np.unique(a, return_inverse=True)
        dev_a = torch.from_numpy(inv.reshape(a.shape).astype(np.int32)).to(require_device())
        E = len(ids)
    else:
        ids = None
        dev_a = table.device_assignment()
    demand = device_histograms(dev_a, E)
    if distinct_only:
        caps, inf = (demand > 0).to(torch.int32), torch.zeros(L, dtype=torch.int32)
    else:
        caps, inf = cap_device(demand, capacity)
    caps, inf = caps.cpu().numpy(), inf.cpu().numpy()
    layers = []
    for l, row in enumerate(caps):
        if inf[l]:
            layers.append({})
            continue
        nz = np.nonzero(row)[0]
        keys = nz if ids is None else ids[nz]
        layers.append({int(e): int(c) for e, c in zip(keys, row[nz])})
    return ReplicaPlan(capacity=capacity, layers=layers)
