"""Per-layer expert residency -- drop-in for ``moesim.placement``
(reference src/placement.py:1-180) plus the execution map of
``BatchRunner._run_predicted`` (src/simulator.py:181-208).

The residency update and the token walk run on the GPU (mp_place: chunked
stable ranks + closed form slot(t) = off[e] + (rank_e(t) + r_e) mod cnt_e,
SURVEY.md F5); the execution map runs in mp_exec_map (F6). Because replica
ordinals are always 0..n-1 (src/placement.py:89-100), a per-expert count is the
whole device state; ``DeviceState`` keeps the reference's dict-of-lists view.
The TransferLog is rebuilt on the host from the per-token event codes and
per-expert offload counts the kernels emit, in the reference's exact order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._dev import WORKSPACE, ptr, require_device, stream_ptr
from .errors import ConfigurationError
from .planner import ReplicaPlan, check_positive
from .predictor import HashTable
from .router_oracle import LayerPlacement, Placement

LOAD = "load"
REPLICATE = "replicate"
OFFLOAD = "offload"


@dataclass(frozen=True)
class TransferEvent:
    kind: str
    layer: int
    expert: int
    ordinal: int


@dataclass
class TransferLog:
    """Ordered transfer events plus the layers that needed the distinct-only fallback (src/placement.py:35-63)."""

    events: list[TransferEvent] = field(default_factory=list)
    fallback_layers: list[int] = field(default_factory=list)

    def record(self, kind: str, layer: int, expert: int, ordinal: int) -> None:
        self.events.append(TransferEvent(kind, layer, expert, ordinal))

    def count(self, kind: str) -> int:
        return sum(1 for e in self.events if e.kind == kind)

    def layer_events(self, layer: int) -> list[TransferEvent]:
        return [e for e in self.events if e.layer == layer]

    def extend(self, other: "TransferLog") -> None:
        self.events.extend(other.events)
        self.fallback_layers.extend(other.fallback_layers)

    def to_csv_rows(self):
        for seq, e in enumerate(self.events):
            yield {"event": e.kind, "layer": e.layer, "expert": e.expert, "ordinal": e.ordinal, "sequence": seq}


class DeviceState:
    """Resident replica slots per layer, capped at ``capacity`` slots each (src/placement.py:66-100)."""

    def __init__(self, num_layers: int, capacity: int):
        self.num_layers = check_positive("num_layers", num_layers)
        self.capacity = check_positive("capacity", capacity)
        self._resident: list[dict[int, list[int]]] = [{} for _ in range(num_layers)]
        self.last_place_device = None  # device arrays of the last apply_batch / execution_map
        self.last_exec_device = None   # (cost-model counts, simulator.py)

    def resident(self, layer: int) -> dict[int, list[int]]:
        return self._resident[layer]

    def resident_slot_count(self, layer: int) -> int:
        return sum(len(o) for o in self._resident[layer].values())

    def slots(self, layer: int) -> list[tuple[int, int]]:
        """Resident slots in deterministic (expert, ordinal) order."""
        return sorted((e, o) for e, ords in self._resident[layer].items() for o in ords)

    def add_replica(self, layer: int, expert: int) -> int:
        ords = self._resident[layer].setdefault(expert, [])
        o = ords[-1] + 1 if ords else 0
        ords.append(o)
        return o

    def drop_replica(self, layer: int, expert: int) -> int:
        ords = self._resident[layer][expert]
        o = ords.pop()
        if not ords:
            del self._resident[layer][expert]
        return o

    # -- dense views used by the kernels -------------------------------------------------
    def counts(self, layer: int, ids: np.ndarray) -> np.ndarray:
        pos = {int(e): i for i, e in enumerate(ids)}
        out = np.zeros(len(ids), dtype=np.int32)
        for e, ords in self._resident[layer].items():
            out[pos[e]] = len(ords)
        return out

    def set_counts(self, layer: int, ids: np.ndarray, counts: np.ndarray) -> None:
        res = self._resident[layer]
        res.clear()
        for i in np.nonzero(counts)[0]:
            res[int(ids[i])] = list(range(int(counts[i])))


def _layer_caps(plan: ReplicaPlan, layer: int) -> dict[int, int]:
    if layer >= len(plan.layers):
        raise ConfigurationError(f"plan covers {len(plan.layers)} layers, needed layer {layer}")
    return plan.layers[layer]


def _id_space(rows: np.ndarray, extra: list) -> np.ndarray:
    """Sorted expert ids the kernels index densely (order preserving)."""
    keys = set()
    for d in extra:
        keys.update(int(k) for k in d)
    mx = max([int(rows.max()) if rows.size else -1] + [k for k in keys] + [-1])
    if mx < (1 << 16):
        return np.arange(mx + 1, dtype=np.int64)
    return np.union1d(np.unique(rows), np.array(sorted(keys), dtype=np.int64))


def _place_layers(state: DeviceState, rows: np.ndarray, layers: list[int], caps_list: list[dict],
                  plan_capacity: int, log: TransferLog) -> list[np.ndarray]:
    """Run mp_place over the given layers (in order); update state and log; return token maps."""
    dev = require_device()
    L, T = len(layers), rows.shape[1]
    ids = _id_space(rows, caps_list + [state.resident(l) for l in layers])
    E = max(len(ids), 1)
    dense = {int(e): i for i, e in enumerate(ids)} if len(ids) and ids[-1] != len(ids) - 1 else None
    a = rows if dense is None else np.vectorize(dense.__getitem__, otypes=[np.int64])(rows)
    caps = np.zeros((L, E), dtype=np.int32)
    res = np.zeros((L, E), dtype=np.int32)
    for i, l in enumerate(layers):
        for e, c in caps_list[i].items():
            caps[i, int(e) if dense is None else dense[int(e)]] = int(c)
        res[i] = state.counts(l, ids) if len(ids) else 0
    a_d = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)
    caps_d = torch.from_numpy(caps).to(dev)
    res_d = torch.from_numpy(res).to(dev)
    i32 = dict(dtype=torch.int32, device=dev)
    tts = torch.empty(L, max(T, 1), **i32)
    tev = torch.empty(L, max(T, 1), **i32)
    offl = torch.empty(L, E, **i32)
    fb = torch.empty(L, **i32)
    ns = torch.empty(L, **i32)
    nbytes = _lib.size_query("mp_place_workspace_bytes", L, T, E)
    ws = WORKSPACE.get("place", nbytes, dev)
    _lib.call("mp_place", ptr(a_d), L, T, E, ptr(caps_d), int(plan_capacity), int(state.capacity), ptr(res_d),
              ptr(tts), ptr(tev), ptr(offl), ptr(fb), ptr(ns), ptr(ws), nbytes, stream_ptr())
    # device-side results of the last placement, for the cost-model counts (simulator.py)
    state.last_place_device = {"layers": list(layers), "token_event": tev, "offloads": offl, "E": E, "T": T}
    tts, tev, offl, fb, res_new = (t.cpu().numpy() for t in (tts, tev, offl, fb, res_d))
    out = []
    for i, l in enumerate(layers):
        # reclaim pops (demanded experts, ascending), then full offloads of the rest
        # (src/placement.py:133-141); a demanded expert keeps >= 1 resident slot.
        res_prev = res[i]
        for j in np.nonzero((offl[i] > 0) & (res_new[i] > 0))[0]:
            for o in range(res_prev[j] - 1, res_prev[j] - 1 - offl[i, j], -1):
                log.record(OFFLOAD, l, int(ids[j]), int(o))
        for j in np.nonzero((offl[i] > 0) & (res_new[i] == 0))[0]:
            for o in range(res_prev[j] - 1, -1, -1):
                log.record(OFFLOAD, l, int(ids[j]), int(o))
        ev = tev[i, :T]
        for t in np.nonzero(ev >= 0)[0]:
            kind = LOAD if (ev[t] >> _lib.MP_EVENT_KIND_SHIFT) == _lib.MP_EVENT_LOAD else REPLICATE
            log.record(kind, l, int(rows[i, t]), int(ev[t] & ((1 << _lib.MP_EVENT_KIND_SHIFT) - 1)))
        if fb[i]:
            log.fallback_layers.append(l)
        state.set_counts(l, ids, res_new[i])
        out.append(tts[i, :T].astype(np.int64))
    return out


def apply_layer(state: DeviceState, table: HashTable, plan: ReplicaPlan, layer: int):
    """Place one layer of a hash table; returns (state, token_to_slot, TransferLog) (src/placement.py:109-165).

    The device state is updated in place. The returned token map indexes into
    ``state.slots(layer)`` taken after placement.
    """
    caps = _layer_caps(plan, layer)
    log = TransferLog()
    rows = table.assignment[layer: layer + 1]
    (tts,) = _place_layers(state, rows, [layer], [caps], plan.capacity, log)
    return state, tts, log


def apply_batch(state: DeviceState, table: HashTable, plan: ReplicaPlan):
    """Fold apply_layer over every layer; returns (state, Placement, TransferLog) (src/placement.py:168-180)."""
    if table.num_layers != state.num_layers:
        raise ConfigurationError(f"table has {table.num_layers} layers, device has {state.num_layers}")
    log = TransferLog()
    n = min(table.num_layers, len(plan.layers))
    layers = []
    if n:
        maps = _place_layers(state, table.assignment[:n], list(range(n)), plan.layers[:n], plan.capacity, log)
        layers = [LayerPlacement(slots=state.slots(l), token_to_slot=m) for l, m in enumerate(maps)]
    if n < table.num_layers:
        _layer_caps(plan, n)  # raises ConfigurationError like the reference's sequential fold
    return state, Placement(layers=layers), log


def execution_map(state: DeviceState, true_routing):
    """Map tokens onto replicas of their TRUE expert (src/simulator.py:185-203).

    Every expert routed to but not resident gets one corrective LOAD (ordinal 0,
    persisted in ``state``); tokens of an expert round-robin over its resident
    replicas in token order. Returns (state, Placement, TransferLog).
    """
    dev = require_device()
    rows = np.asarray(true_routing, dtype=np.int64)
    if rows.ndim != 2 or rows.shape[0] != state.num_layers:
        raise ConfigurationError(f"routing must be ({state.num_layers}, tokens)")
    L, T = rows.shape
    log = TransferLog()
    if T == 0:
        return state, Placement([LayerPlacement(state.slots(l), np.zeros(0, np.int64)) for l in range(L)]), log
    ids = _id_space(rows, [state.resident(l) for l in range(L)])
    E = len(ids)
    dense = {int(e): i for i, e in enumerate(ids)} if ids[-1] != E - 1 else None
    a = rows if dense is None else np.vectorize(dense.__getitem__, otypes=[np.int64])(rows)
    res = np.stack([state.counts(l, ids) for l in range(L)])
    max_slots = int(res.sum(axis=1).max()) + E
    i32 = dict(dtype=torch.int32, device=dev)
    a_d = torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)
    res_d = torch.from_numpy(res).to(dev)
    tts = torch.empty(L, T, **i32)
    corr = torch.empty(L, E, **i32)
    ns = torch.empty(L, **i32)
    tor = torch.empty(L, T, **i32)
    pstride = max_slots + (T + 127) // 128
    prow = torch.empty(L, pstride, **i32)
    prows = torch.empty(L, pstride, **i32)
    eb = torch.empty(L, E + 1, **i32)
    nbytes = _lib.size_query("mp_exec_workspace_bytes", L, T, E, max_slots)
    ws = WORKSPACE.get("exec", nbytes, dev)
    _lib.call("mp_exec_map", ptr(a_d), L, T, E, max_slots, 0, ptr(res_d), ptr(tts), ptr(corr), ptr(ns), None,
              ptr(tor), ptr(prow), ptr(prows), ptr(eb), ptr(ws), nbytes, stream_ptr())
    state.last_exec_device = {"token_to_slot": tts, "corrective": corr, "num_slots": ns, "E": E, "T": T,
                              "max_slots": max_slots}
    tts, corr, res_new = tts.cpu().numpy(), corr.cpu().numpy(), res_d.cpu().numpy()
    layers = []
    for l in range(L):
        for j in np.nonzero(corr[l])[0]:
            log.record(LOAD, l, int(ids[j]), 0)
        state.set_counts(l, ids, res_new[l])
        layers.append(LayerPlacement(slots=state.slots(l), token_to_slot=tts[l].astype(np.int64)))
    return state, Placement(layers=layers), log
