"""Top-1 MoE forward -- drop-in for ``moesim.router_oracle``
(reference src/router_oracle.py:1-178), running on sm_100a.

* ``route_top1`` / the dense baseline route with mp_route_top1: split-bf16
  tensor-core logits plus an exact float64 re-decision of near-ties, so the
  chosen experts equal the reference's float64 argmax (lowest index on ties).
* expert FFNs + residual combine run as one grouped tcgen05 GEMM pair over
  replica segments (mp_moe_ffn); replicas alias one weight copy, and each
  token's arithmetic is independent of the segment it lands in, so a
  replicated placement is bitwise equal to the dense baseline on the GPU (the
  GPU analogue of src/router_oracle.py:1-7 / pkg/tests/test_acceptance.py:45-70).
* bf16 operands with fp32 accumulation: max-norm relative error vs the float32
  reference <= 1e-2 (tests/test_parity_gpu.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import WORKSPACE, download, ptr, require_device, round_up, stream_ptr, upload_rows
from .errors import ConfigurationError, PlacementError
from .predictor import check_finite

DENSE_BASELINE = "dense-baseline"


@dataclass
class ToyMoeParams:
    """Router and expert weights for every layer (src/router_oracle.py:22-61).

    router_weights: (L, E, d_model); expert_u: (L, E, d_ff, d_model);
    expert_v: (L, E, d_model, d_ff). All float32.
    """

    router_weights: np.ndarray
    expert_u: np.ndarray
    expert_v: np.ndarray

    def __post_init__(self):
        if self.router_weights.ndim != 3 or self.expert_u.ndim != 4 or self.expert_v.ndim != 4:
            raise ConfigurationError("parameter tensors have wrong rank")
        layers, experts, d_model = self.router_weights.shape
        d_ff = self.expert_u.shape[2]
        if self.expert_u.shape != (layers, experts, d_ff, d_model):
            raise ConfigurationError(f"expert_u shape {self.expert_u.shape} inconsistent")
        if self.expert_v.shape != (layers, experts, d_model, d_ff):
            raise ConfigurationError(f"expert_v shape {self.expert_v.shape} inconsistent")
        check_finite("router_weights", self.router_weights)
        check_finite("expert_u", self.expert_u)
        check_finite("expert_v", self.expert_v)

    @property
    def num_layers(self) -> int:
        return self.router_weights.shape[0]

    @property
    def num_experts(self) -> int:
        return self.router_weights.shape[1]

    @property
    def d_model(self) -> int:
        return self.router_weights.shape[2]

    @property
    def d_ff(self) -> int:
        return self.expert_u.shape[2]


@dataclass
class LayerPlacement:
    """Resident replica slots for one layer plus the token-to-slot assignment (src/router_oracle.py:64-69)."""

    slots: list[tuple[int, int]]
    token_to_slot: np.ndarray


@dataclass
class Placement:
    layers: list[LayerPlacement]


def random_params(shape, d_ff: int | None = None, seed: int = 0) -> ToyMoeParams:
    """Fully random toy model (src/router_oracle.py:77-87; same RNG stream)."""
    if d_ff is None:
        d_ff = shape.d_model
    rng = np.random.default_rng(seed)
    layers, experts, d_model = shape.num_layers, shape.experts_per_layer, shape.d_model
    return ToyMoeParams(
        router_weights=rng.normal(size=(layers, experts, d_model)).astype(np.float32),
        expert_u=rng.normal(0.0, 1.0 / np.sqrt(d_model), size=(layers, experts, d_ff, d_model)).astype(np.float32),
        expert_v=rng.normal(0.0, 1.0 / np.sqrt(d_ff), size=(layers, experts, d_model, d_ff)).astype(np.float32),
    )


# ----------------------------------------------------------------------------- device weights


def router_eg(E: int) -> int:
    for g in (64, 128, 256):
        if E <= g:
            return g
    raise ConfigurationError(f"{E} experts per layer: the router tile supports at most 256")


class DeviceMoeLayer:
    """One MoE layer's weights in kernel layout (d padded to dp % 64, d_ff to Fp % 256):
    router w_hl = [bf16(w) | bf16(w - bf16(w))] (Eg x 2dp), w32 (E x dp) fp32,
    w_abs[k] = max_e |w_ek|; U (E*Fp x dp) bf16, V (E*dp x Fp) bf16."""

    def __init__(self, router: torch.Tensor, u: torch.Tensor, v: torch.Tensor, dp: int, Fp: int):
        dev = router.device
        E, d = router.shape
        F = u.shape[1]
        self.E, self.d, self.F, self.dp, self.Fp = E, d, F, dp, Fp
        self.Eg = router_eg(E)
        w32 = torch.zeros(E, dp, device=dev)
        w32[:, :d] = router.float()
        hi = w32.to(torch.bfloat16)
        lo = (w32 - hi.float()).to(torch.bfloat16)
        self.w_hl = torch.zeros(self.Eg, 2 * dp, device=dev, dtype=torch.bfloat16)
        self.w_hl[:E, :dp] = hi
        self.w_hl[:E, dp:] = lo
        self.w32 = w32
        self.w_abs = torch.empty(dp, device=dev)
        _lib.call("mp_router_weight_absmax", ptr(self.w32), E, dp, ptr(self.w_abs), stream_ptr())
        U = torch.zeros(E, Fp, dp, device=dev, dtype=torch.bfloat16)
        U[:, :F, :d] = u.to(torch.bfloat16)
        V = torch.zeros(E, dp, Fp, device=dev, dtype=torch.bfloat16)
        V[:, :d, :F] = v.to(torch.bfloat16)
        self.U = U.view(E * Fp, dp)
        self.V = V.view(E * dp, Fp)
        self.tiled = 0


class DeviceMoe:
    def __init__(self, params: ToyMoeParams, device: torch.device):
        self.L, self.E, self.d, self.F = params.num_layers, params.num_experts, params.d_model, params.d_ff
        self.dp = round_up(max(self.d, 64), 64)
        self.Fp = round_up(max(self.F, 256), 256)
        self.layers = []
        for l in range(self.L):
            r = torch.from_numpy(np.ascontiguousarray(params.router_weights[l])).to(device)
            u = torch.from_numpy(np.ascontiguousarray(params.expert_u[l])).to(device)
            v = torch.from_numpy(np.ascontiguousarray(params.expert_v[l])).to(device)
            self.layers.append(DeviceMoeLayer(r, u, v, self.dp, self.Fp))


def _device_moe(params: ToyMoeParams, device) -> DeviceMoe:
    key = tuple((id(a), a.__array_interface__["data"][0], a.shape)
                for a in (params.router_weights, params.expert_u, params.expert_v))
    big = params.expert_u.nbytes + params.expert_v.nbytes > (16 << 20)
    cached = getattr(params, "_device_cache", None)
    if big and cached is not None and cached[0] == key:
        return cached[1]
    dm = DeviceMoe(params, device)
    if big:
        object.__setattr__(params, "_device_cache", (key, dm))
    return dm


# ----------------------------------------------------------------------------- device ops


def route_device(x: torch.Tensor, layer: DeviceMoeLayer, stream=None) -> torch.Tensor:
    """(T, dp) fp32 stream -> (T,) int32 top-1 experts (fp64-faithful)."""
    T = x.shape[0]
    route = torch.empty(T, dtype=torch.int32, device=x.device)
    nbytes = _lib.size_query("mp_router_workspace_bytes", T, layer.dp)
    ws = WORKSPACE.get("router", nbytes, x.device)
    _lib.call("mp_route_top1_ex", ptr(x), layer.dp, T, layer.dp, ptr(layer.w_hl), ptr(layer.w32), ptr(layer.w_abs),
              layer.E, layer.Eg, ptr(route), ptr(ws), nbytes, stream_ptr(stream))
    return route


def segments_device(token_to_slot: torch.Tensor, slot_expert: torch.Tensor, E: int, split_m: int = 1, stream=None):
    """Slot-grouped row permutation + GEMM pieces from a token -> slot map (slots sorted by expert)."""
    T = token_to_slot.shape[0]
    S = slot_expert.shape[0]
    dev = token_to_slot.device
    i32 = dict(dtype=torch.int32, device=dev)
    tor = torch.empty(T, **i32)
    pn = S + (T + 127) // 128
    prow = torch.empty(pn, **i32)
    prows = torch.empty(pn, **i32)
    eb = torch.empty(E + 1, **i32)
    nbytes = _lib.size_query("mp_segments_workspace_bytes", T, S)
    ws = WORKSPACE.get("segments", nbytes, dev)
    _lib.call("mp_segments_from_slots", ptr(token_to_slot), ptr(slot_expert), T, S, E, split_m, ptr(tor), ptr(prow),
              ptr(prows), ptr(eb), ptr(ws), nbytes, stream_ptr(stream))
    return tor, prow, prows, eb


def ffn_device(x: torch.Tensor, y: torch.Tensor, layer: DeviceMoeLayer, tor, prow, prows, eb, stream=None):
    """y[tok] += V_e relu(U_e x[tok]) over the given segments (y is x for the residual stream)."""
    T = x.shape[0]
    nbytes = _lib.size_query("mp_ffn_workspace_bytes", T, layer.dp, layer.Fp)
    ws = WORKSPACE.get("ffn", nbytes, x.device)
    _lib.call("mp_moe_ffn", ptr(x), ptr(y), T, layer.dp, layer.Fp, layer.E, ptr(layer.U), ptr(layer.V), ptr(tor),
              ptr(prow), ptr(prows), ptr(eb), ptr(ws), nbytes, stream_ptr(stream))


def _stream_device(embeddings, d: int, dp: int, dev) -> torch.Tensor:
    emb = getattr(embeddings, "embeddings", embeddings)
    x = upload_rows(emb, d, dp, dev)
    if x.ndim != 2 or x.shape[1] != dp:
        raise ConfigurationError(f"embeddings shape {tuple(np.shape(emb))} != (tokens, {d})")
    return x


# ----------------------------------------------------------------------------- public API


def route_top1(layer: int, embedding, params: ToyMoeParams) -> int:
    """Argmax of the layer's router logits; ties break toward the lower index (src/router_oracle.py:90-98)."""
    if layer < 0 or layer >= params.num_layers:
        raise ConfigurationError(f"layer {layer} outside [0, {params.num_layers})")
    emb = check_finite("embedding", embedding).astype(np.float64)
    if emb.shape != (params.d_model,):
        raise ConfigurationError(f"embedding shape {emb.shape} != ({params.d_model},)")
    dev = require_device()
    dm = _device_moe(params, dev)
    x = _stream_device(emb.astype(np.float32)[None, :], params.d_model, dm.dp, dev)
    return int(route_device(x, dm.layers[layer])[0].item())


def expert_forward(embedding, u, v) -> np.ndarray:
    """One expert FFN: v @ relu(u @ x) (src/router_oracle.py:101-111)."""
    emb = check_finite("embedding", embedding)
    u = np.asarray(u)
    v = np.asarray(v)
    if u.ndim != 2 or v.ndim != 2 or u.shape[1] != emb.shape[-1] or v.shape[1] != u.shape[0]:
        raise ConfigurationError(f"incompatible expert shapes u={u.shape} v={v.shape} x={emb.shape}")
    dev = require_device()
    d, F = u.shape[1], u.shape[0]
    dp, Fp = round_up(max(d, 64), 64), round_up(max(F, 256), 256)
    zero_router = torch.zeros(1, d, device=dev)
    lay = DeviceMoeLayer(zero_router, torch.from_numpy(np.asarray(u, np.float32))[None].to(dev),
                         torch.from_numpy(np.asarray(v, np.float32))[None].to(dev), dp, Fp)
    x = _stream_device(np.asarray(emb, np.float32)[None, :], d, dp, dev)
    y = torch.zeros_like(x)
    zero = torch.zeros(1, dtype=torch.int32, device=dev)
    tor, prow, prows, eb = segments_device(zero, zero, 1)
    ffn_device(x, y, lay, tor, prow, prows, eb)
    out = y[0, : v.shape[0]].cpu().numpy()
    return check_finite("expert output", out)


def _run_layers_device(x: torch.Tensor, dm: DeviceMoe, placement=None, record=False):
    """Shared forward loop (src/router_oracle.py:119-135): route or look up the slot's expert,
    grouped expert FFN, residual combine. Returns chosen experts (L, T) when record."""
    T = x.shape[0]
    chosen = []
    arange_e = torch.arange(dm.E, dtype=torch.int32, device=x.device)
    for l, lay in enumerate(dm.layers):
        if placement is None:
            route = route_device(x, lay)
            tor, prow, prows, eb = segments_device(route, arange_e, dm.E)
            if record:
                chosen.append(route)
        else:
            tts, slot_expert = placement[l]
            tor, prow, prows, eb = segments_device(tts, slot_expert, dm.E)
        ffn_device(x, x, lay, tor, prow, prows, eb)
    return chosen


def oracle_route_batch(batch, params: ToyMoeParams) -> np.ndarray:
    """(L, B) expert indices the dense model itself picks, layer by layer (src/router_oracle.py:138-142)."""
    dev = require_device()
    dm = _device_moe(params, dev)
    x = _stream_device(batch, params.d_model, dm.dp, dev)
    if x.shape[0] == 0:
        return np.zeros((params.num_layers, 0), dtype=np.int64)
    chosen = _run_layers_device(x, dm, record=True)
    return torch.stack(chosen).cpu().numpy().astype(np.int64)


def _validated_placement(placement: Placement, params: ToyMoeParams, T: int, dev):
    """Reference checks of moe_forward's choose() (src/router_oracle.py:165-175), in the same
    layer-then-token order; slots re-indexed so slot experts are non-decreasing."""
    if len(placement.layers) != params.num_layers:
        raise PlacementError(
            f"placement covers {len(placement.layers)} layers, model has {params.num_layers}"
        )
    out = []
    for layer, lp in enumerate(placement.layers):
        tts = np.asarray(lp.token_to_slot, dtype=np.int64)
        if tts.shape[0] < T:
            raise PlacementError(f"layer {layer}: no slot assigned to token {tts.shape[0]}")
        tts = tts[:T]
        nslots = len(lp.slots)
        slot_expert = np.array([s[0] for s in lp.slots], dtype=np.int64)
        ok_slot = (tts >= 0) & (tts < nslots)
        exp_t = np.where(ok_slot, slot_expert[np.clip(tts, 0, max(nslots - 1, 0))] if nslots else -1, -1)
        ok = ok_slot & (exp_t >= 0) & (exp_t < params.num_experts)
        if not ok.all():
            t = int(np.nonzero(~ok)[0][0])
            if not ok_slot[t]:
                raise PlacementError(f"layer {layer}: token {t} mapped to missing slot {int(tts[t])}")
            raise PlacementError(f"layer {layer}: slot {int(tts[t])} holds invalid expert {int(exp_t[t])}")
        order = np.argsort(slot_expert, kind="stable")
        newpos = np.empty_like(order)
        newpos[order] = np.arange(len(order))
        out.append((torch.from_numpy(newpos[tts].astype(np.int32)).to(dev),
                    torch.from_numpy(slot_expert[order].astype(np.int32)).to(dev)))
    return out


def moe_forward(batch, params: ToyMoeParams, placement=DENSE_BASELINE) -> np.ndarray:
    """Run the toy MoE over a batch and return the (B, d_model) final stream (src/router_oracle.py:145-178).

    With ``placement="dense-baseline"`` every layer routes via route_top1 with all
    experts available. With a Placement, each token uses the logical expert of its
    assigned slot; replicas alias one weight copy, so the output equals the baseline
    bit for bit whenever the placement follows the model's routing.
    """
    dev = require_device()
    if isinstance(placement, str):
        if placement != DENSE_BASELINE:
            raise ConfigurationError(f"unknown placement mode {placement!r}")
    dm = _device_moe(params, dev)
    x = _stream_device(batch, params.d_model, dm.dp, dev)
    T = x.shape[0]
    if T == 0:
        return np.zeros((0, params.d_model), dtype=np.float32)
    if isinstance(placement, str):
        _run_layers_device(x, dm)
    else:
        _run_layers_device(x, dm, placement=_validated_placement(placement, params, T, dev))
    return download(x[:, : params.d_model] if params.d_model != dm.dp else x)


# ---------------------------------------------------------------- parameter files
PARAMS_FORMAT_VERSION = "1"


def save_params(params: ToyMoeParams, path) -> None:
    """``moesim-moe-params v1`` (src/router_oracle.py:184-206): one float32 tensor row per line."""
    from .workload import fmt_f32

    out = [f"moesim-moe-params v{PARAMS_FORMAT_VERSION} layers={params.num_layers} experts={params.num_experts} "
           f"d_model={params.d_model} d_ff={params.d_ff}"]
    for name, t in (("router", params.router_weights), ("expert_u", params.expert_u), ("expert_v", params.expert_v)):
        out.extend(name + " " + " ".join(fmt_f32(v) for v in row) for row in t.reshape(-1, t.shape[-1]))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(out) + "\n")


def load_params(path) -> ToyMoeParams:
    """Inverse of save_params (src/router_oracle.py:209-251), same TraceParseError cases."""
    from .errors import TraceParseError
    from .workload import parse_param_header, read_rows

    with open(path, encoding="utf-8") as fh:
        h = parse_param_header(fh.readline(), "moesim-moe-params", ("layers", "experts", "d_model", "d_ff"))
        L, E, d, F = h["layers"], h["experts"], h["d_model"], h["d_ff"]
        ln = [1]
        t = {}
        for name, shape, width in (("router", (L, E, d), d), ("expert_u", (L, E, F, d), d),
                                   ("expert_v", (L, E, d, F), F)):
            t[name] = read_rows(fh, name, int(np.prod(shape[:-1])), width, ln, np.float32).reshape(shape)
        if fh.readline():
            raise TraceParseError("trailing data after parameter rows", line=ln[0] + 1)
    return ToyMoeParams(router_weights=t["router"], expert_u=t["expert_u"], expert_v=t["expert_v"])


def load_params_device(path, device=None) -> "DeviceMoe":
    """load_params + the device layout the kernels use (split-bf16 router, bf16 K-major experts)."""
    return _device_moe(load_params(path), device or require_device())
