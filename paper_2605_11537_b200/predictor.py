"""SRU expert predictor and hash-table construction -- drop-in for
``moesim.predictor`` (reference src/predictor.py:1-232), running on sm_100a.

Same names, signatures, dataclasses and exceptions as the reference. The
arithmetic runs in libmoempmc.so:
  * ``sru_forward`` / ``sru_cell``  -> mp_sru_layer (tcgen05 projection GEMM +
    chunked scan), bf16 operands, fp32 accumulation and state;
  * ``predict_batch``               -> mp_sru_layer x S, mp_heads_argmax
    (argmax of the head logits == argmax of their sparsemax);
  * ``HashTable`` histograms        -> mp_histogram;
  * ``sparsemax``                   -> mp_sparsemax_rows (float64).
Outputs are returned as numpy like the reference. Tolerance vs the float64
reference: max-norm relative error <= 1e-2 on hidden states (bf16 operands);
predicted-expert argmax flips are counted by the parity tests.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from ._dev import WORKSPACE, download, pow2_at_least, ptr, require_device, round_up, stream_ptr, upload_rows
from .errors import ConfigurationError, NumericError

DEFAULT_SRU_LAYERS = 10  # src/predictor.py:19


def check_finite(name: str, arr) -> np.ndarray:
    """src/validation.py:22-27."""
    arr = np.asarray(arr)
    if not np.all(np.isfinite(arr)):
        raise NumericError(f"{name} contains non-finite values")
    return arr


@dataclass
class SruLayerParams:
    """Weights of one SRU layer: w, w_f, w_r are (d, d); b_f, b_r are (d,) (src/predictor.py:28-36)."""

    w: np.ndarray
    w_f: np.ndarray
    w_r: np.ndarray
    b_f: np.ndarray
    b_r: np.ndarray


@dataclass
class SruParams:
    """SRU trunk shared by all MoE layers plus one (E, d) head per MoE layer (src/predictor.py:39-69)."""

    layers: list[SruLayerParams]
    heads: np.ndarray  # (num_moe_layers, E, d_model)

    @property
    def num_sru_layers(self) -> int:
        return len(self.layers)

    @property
    def num_moe_layers(self) -> int:
        return self.heads.shape[0]

    @property
    def num_experts(self) -> int:
        return self.heads.shape[1]

    @property
    def d_model(self) -> int:
        return self.heads.shape[2]

    def copy(self) -> "SruParams":
        return SruParams(
            layers=[
                SruLayerParams(l.w.copy(), l.w_f.copy(), l.w_r.copy(), l.b_f.copy(), l.b_r.copy())
                for l in self.layers
            ],
            heads=self.heads.copy(),
        )


@dataclass
class SruState:
    """Cell state per SRU layer; zeros at the start of every batch (src/predictor.py:72-80)."""

    cells: np.ndarray

    @classmethod
    def zeros(cls, num_sru_layers: int, d_model: int) -> "SruState":
        return cls(np.zeros((num_sru_layers, d_model)))


def device_histograms(assign_dev: torch.Tensor, num_experts: int) -> torch.Tensor:
    """(L, T) int32 device assignment -> (L, E) int32 demand via mp_histogram."""
    L, T = assign_dev.shape
    out = torch.empty(L, num_experts, dtype=torch.int32, device=assign_dev.device)
    _lib.call("mp_histogram", ptr(assign_dev), L, T, num_experts, ptr(out), stream_ptr())
    return out


def _histograms(assignment: np.ndarray, device_copy: torch.Tensor | None = None) -> list[dict[int, int]]:
    """src/predictor.py:122-127 on the GPU: expert -> count per layer row."""
    if assignment.size == 0:
        return [{} for _ in range(assignment.shape[0])]
    dev = require_device()
    E = int(assignment.max()) + 1
    if E > 1 << 16:  # sparse ids: histogram over the compressed id space (order preserving)
        ids, inv = np.unique(assignment, return_inverse=True)
        a = torch.from_numpy(inv.reshape(assignment.shape).astype(np.int32)).to(dev)
        counts = device_histograms(a, len(ids)).cpu().numpy()
    else:
        ids = None
        a = device_copy if device_copy is not None else torch.from_numpy(assignment.astype(np.int32)).to(dev)
        counts = device_histograms(a, E).cpu().numpy()
    out = []
    for row in counts:
        nz = np.nonzero(row)[0]
        keys = nz if ids is None else ids[nz]
        out.append({int(e): int(c) for e, c in zip(keys, row[nz])})
    return out


@dataclass
class HashTable:
    """Predicted (layer, token) -> expert map plus per-expert replica demand (src/predictor.py:83-119)."""

    batch_index: int
    assignment: np.ndarray  # (num_moe_layers, batch_size) int64
    replica_counts: list[dict[int, int]] = field(default_factory=list)
    _device: torch.Tensor | None = field(default=None, repr=False, compare=False)

    def __post_init__(self):
        if self.assignment.ndim != 2:
            raise ConfigurationError("assignment must be (layers, tokens)")
        if self.assignment.size and self.assignment.min() < 0:
            raise ConfigurationError("assignment holds negative expert indices")
        expected = _histograms(self.assignment, self._device)
        if not self.replica_counts:
            self.replica_counts = expected
        elif self.replica_counts != expected:
            raise ConfigurationError("replica_counts do not match the assignment histogram")

    @classmethod
    def from_assignment(cls, batch_index: int, assignment) -> "HashTable":
        return cls(batch_index, np.asarray(assignment, dtype=np.int64))

    @property
    def num_layers(self) -> int:
        return self.assignment.shape[0]

    @property
    def num_tokens(self) -> int:
        return self.assignment.shape[1]

    def device_assignment(self) -> torch.Tensor:
        """(L, T) int32 copy on the GPU (cached when produced by predict_batch)."""
        if self._device is None:
            self._device = torch.from_numpy(self.assignment.astype(np.int32)).to(require_device())
        return self._device

    def __eq__(self, other):
        if not isinstance(other, HashTable):
            return NotImplemented
        return self.batch_index == other.batch_index and np.array_equal(self.assignment, other.assignment)


def init_params(
    num_moe_layers: int,
    num_experts: int,
    d_model: int,
    num_sru_layers: int = DEFAULT_SRU_LAYERS,
    seed: int = 0,
) -> SruParams:
    """Seeded uniform init in [-1/sqrt(d), 1/sqrt(d)], draw order w, w_f, w_r, b_f, b_r per
    layer then heads -- identical values to src/predictor.py:130-154 (host-side setup)."""
    rng = np.random.default_rng(seed)
    bound = 1.0 / np.sqrt(d_model)

    def draw(*shape):
        return rng.uniform(-bound, bound, size=shape)

    layers = [
        SruLayerParams(w=draw(d_model, d_model), w_f=draw(d_model, d_model), w_r=draw(d_model, d_model),
                       b_f=draw(d_model), b_r=draw(d_model))
        for _ in range(num_sru_layers)
    ]
    return SruParams(layers=layers, heads=draw(num_moe_layers, num_experts, d_model))


# ----------------------------------------------------------------------------- device weights


class DeviceSru:
    """SRU + heads weights laid out for the kernels (padded to d % 64 == 0):
    W_cat = [W; W_f; W_r] (3dp x dp bf16, K-major), b_cat = [0; b_f; b_r] fp32,
    heads (ceil64(L*Eg) x dp bf16), layer l in rows [l*Eg, l*Eg + E)."""

    def __init__(self, layers, heads: np.ndarray, device: torch.device):
        d = heads.shape[2] if heads is not None else layers[0][0].shape[0]
        self.d = d
        self.dp = round_up(max(d, 64), 64)
        dp = self.dp
        self.w_cat = []
        self.b_cat = []
        for w, w_f, w_r, b_f, b_r in layers:
            W = torch.zeros(3 * dp, dp, dtype=torch.float32)
            B = torch.zeros(3 * dp, dtype=torch.float32)
            for i, m in enumerate((w, w_f, w_r)):
                W[i * dp: i * dp + d, :d] = torch.as_tensor(np.asarray(m, dtype=np.float64), dtype=torch.float32)
            B[dp: dp + d] = torch.as_tensor(np.asarray(b_f, dtype=np.float64), dtype=torch.float32)
            B[2 * dp: 2 * dp + d] = torch.as_tensor(np.asarray(b_r, dtype=np.float64), dtype=torch.float32)
            self.w_cat.append(W.to(device=device, dtype=torch.bfloat16))
            self.b_cat.append(B.to(device))
        if heads is not None:
            L, E, _ = heads.shape
            self.L, self.E = L, E
            self.Eg = pow2_at_least(E, 32)
            H = torch.zeros(round_up(L * self.Eg, 64), dp, dtype=torch.float32)
            hv = torch.as_tensor(np.asarray(heads, dtype=np.float64), dtype=torch.float32)
            for l in range(L):
                H[l * self.Eg: l * self.Eg + E, :d] = hv[l]
            self.heads = H.to(device=device, dtype=torch.bfloat16)

    @staticmethod
    def from_params(params: SruParams, device: torch.device) -> "DeviceSru":
        layers = [(l.w, l.w_f, l.w_r, l.b_f, l.b_r) for l in params.layers]
        return DeviceSru(layers, params.heads, device)


def _device_sru(params: SruParams, device) -> DeviceSru:
    """Device copy of the predictor weights; cached on the params object when large."""
    nbytes = sum(l.w.nbytes * 3 for l in params.layers) + params.heads.nbytes
    key = tuple((id(a), a.__array_interface__["data"][0], a.shape) for l in params.layers
                for a in (l.w, l.w_f, l.w_r, l.b_f, l.b_r)) + ((id(params.heads), params.heads.shape),)
    cached = getattr(params, "_device_cache", None)
    if nbytes > (8 << 20) and cached is not None and cached[0] == key:
        return cached[1]
    dw = DeviceSru.from_params(params, device)
    if nbytes > (8 << 20):
        object.__setattr__(params, "_device_cache", (key, dw))
    return dw


def sru_stack_device(x32: torch.Tensor, dw: DeviceSru, c0: torch.Tensor | None = None,
                     c_last: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None):
    """Run every SRU layer on a (T, dp) fp32 device sequence; returns (h_f32, h_bf16).

    c0 / c_last: optional (S, dp) cell states entering token 0 / after the last token."""
    T, dp = x32.shape
    dev = x32.device
    sp = stream_ptr(stream)
    nbytes = _lib.size_query("mp_sru_workspace_bytes", T, dp)
    ws = WORKSPACE.get("sru", nbytes, dev)
    nonfinite = torch.zeros(1, dtype=torch.int32, device=dev)
    cur32 = x32
    cur16 = x32.to(torch.bfloat16)
    bufs = [(torch.empty(T, dp, device=dev), torch.empty(T, dp, device=dev, dtype=torch.bfloat16)) for _ in range(2)]
    for i, (W, B) in enumerate(zip(dw.w_cat, dw.b_cat)):
        h32, h16 = bufs[i % 2]
        _lib.call("mp_sru_layer", ptr(cur16), ptr(cur32), ptr(W), ptr(B), T, dp,
                  ptr(c0[i]) if c0 is not None else None, ptr(h32), ptr(h16),
                  ptr(c_last[i]) if c_last is not None else None, ptr(nonfinite), ptr(ws), nbytes, sp)
        cur32, cur16 = h32, h16
    return cur32, cur16, nonfinite


def _embeddings_device(embeddings, d_model: int, dev) -> torch.Tensor:
    x = upload_rows(embeddings, d_model, round_up(max(d_model, 64), 64), dev)
    if x.ndim != 2:
        raise ConfigurationError("embeddings must be (tokens, d_model)")
    if x.shape[0] == 0:
        raise ConfigurationError("batch must contain at least one token")
    if x.shape[1] != round_up(max(d_model, 64), 64):
        raise ConfigurationError(f"embedding width {x.shape[1]} != d_model {d_model}")
    return x


def _raise_if_nonfinite(flag: torch.Tensor) -> None:
    if int(flag.item()) != 0:
        raise NumericError("SRU cell produced non-finite state")


def sru_cell(x_t, c_prev, layer: SruLayerParams):
    """One SRU step (src/predictor.py:157-172); returns (h_t, c_t) float64 arrays."""
    x_t = check_finite("x_t", x_t).astype(np.float64)
    c_prev = check_finite("c_prev", c_prev).astype(np.float64)
    dev = require_device()
    d = x_t.shape[0]
    dw = DeviceSru([(layer.w, layer.w_f, layer.w_r, layer.b_f, layer.b_r)], None, dev)
    x = torch.zeros(1, dw.dp, dtype=torch.float32)
    x[0, :d] = torch.from_numpy(x_t)
    c0 = torch.zeros(1, dw.dp, dtype=torch.float32)
    c0[0, :d] = torch.from_numpy(c_prev)
    x, c0 = x.to(dev), c0.to(dev)
    c_last = torch.zeros(1, dw.dp, device=dev)
    h, _, nf = sru_stack_device(x, dw, c0=c0, c_last=c_last)
    _raise_if_nonfinite(nf)
    return h[0, :d].double().cpu().numpy(), c_last[0, :d].double().cpu().numpy()


def sru_forward(embeddings, params: SruParams) -> np.ndarray:
    """Run the SRU stack over one token sequence; returns (T, d_model) hiddens (src/predictor.py:175-195)."""
    dev = require_device()
    x = _embeddings_device(embeddings, params.d_model, dev)
    dw = _device_sru(params, dev)
    h, _, nf = sru_stack_device(x, dw)
    _raise_if_nonfinite(nf)
    return download(h[:, : params.d_model].double())


def sparsemax(z) -> np.ndarray:
    """Euclidean projection of z onto the probability simplex (src/predictor.py:198-209)."""
    z = check_finite("z", z).astype(np.float64)
    if z.ndim != 1 or z.size == 0:
        raise ConfigurationError("sparsemax expects a nonempty 1-D vector")
    dev = require_device()
    zt = torch.from_numpy(z).to(dev).view(1, -1)
    out = torch.empty_like(zt)
    _lib.call("mp_sparsemax_rows", ptr(zt), 1, z.size, ptr(out), stream_ptr())
    return out[0].cpu().numpy()


def predict_assignment_device(x32: torch.Tensor, dw: DeviceSru, stream=None):
    """(T, dp) fp32 device embeddings -> ((L, T) int32 assignment, nonfinite flag)."""
    T = x32.shape[0]
    _, h16, nf = sru_stack_device(x32, dw, stream=stream)
    assign = torch.empty(dw.L, T, dtype=torch.int32, device=x32.device)
    _lib.call("mp_heads_argmax", ptr(h16), ptr(dw.heads), T, dw.dp, dw.L, dw.E, dw.Eg, ptr(assign),
              stream_ptr(stream))
    return assign, nf


def predict_batch(batch, params: SruParams) -> HashTable:
    """Predict per-layer expert assignments for a batch and count replica demand (src/predictor.py:212-223)."""
    embeddings = getattr(batch, "embeddings", batch)
    index = int(getattr(batch, "index", 0))
    dev = require_device()
    x = _embeddings_device(embeddings, params.d_model, dev)
    dw = _device_sru(params, dev)
    assign, nf = predict_assignment_device(x, dw)
    _raise_if_nonfinite(nf)
    return HashTable(index, assign.cpu().numpy().astype(np.int64), _device=assign)


def evaluate_accuracy(predicted, oracle) -> float:
    """Fraction of (layer, token) cells where the prediction matches the oracle (src/predictor.py:226-232)."""
    pred = predicted.assignment if isinstance(predicted, HashTable) else np.asarray(predicted)
    oracle = np.asarray(oracle)
    if pred.shape != oracle.shape:
        raise ConfigurationError(f"shape mismatch: predicted {pred.shape} vs oracle {oracle.shape}")
    return float(np.mean(pred == oracle))


# ---------------------------------------------------------------- parameter files
SRU_PARAMS_FORMAT_VERSION = "1"


def save_sru_params(params: SruParams, path) -> None:
    """``moesim-sru-params v1`` (src/predictor.py:400-420): float64 rows, 17 significant digits."""
    from .workload import fmt_f64

    out = [f"moesim-sru-params v{SRU_PARAMS_FORMAT_VERSION} sru_layers={params.num_sru_layers} "
           f"moe_layers={params.num_moe_layers} experts={params.num_experts} d_model={params.d_model}"]
    for i, lay in enumerate(params.layers):
        for tag, t in (("w", lay.w), ("wf", lay.w_f), ("wr", lay.w_r), ("bf", lay.b_f.reshape(1, -1)),
                       ("br", lay.b_r.reshape(1, -1))):
            out.extend(f"{tag}{i} " + " ".join(fmt_f64(v) for v in row) for row in t)
    for l in range(params.num_moe_layers):
        out.extend(f"head{l} " + " ".join(fmt_f64(v) for v in row) for row in params.heads[l])
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(out) + "\n")


def load_sru_params(path) -> SruParams:
    """Inverse of save_sru_params (src/predictor.py:423-468), same TraceParseError cases."""
    from .errors import TraceParseError
    from .workload import parse_param_header, read_rows

    with open(path, encoding="utf-8") as fh:
        h = parse_param_header(fh.readline(), "moesim-sru-params", ("sru_layers", "moe_layers", "experts", "d_model"))
        d = h["d_model"]
        ln = [1]
        layers = [SruLayerParams(w=read_rows(fh, f"w{i}", d, d, ln), w_f=read_rows(fh, f"wf{i}", d, d, ln),
                                 w_r=read_rows(fh, f"wr{i}", d, d, ln), b_f=read_rows(fh, f"bf{i}", 1, d, ln)[0],
                                 b_r=read_rows(fh, f"br{i}", 1, d, ln)[0])
                  for i in range(h["sru_layers"])]
        heads = np.stack([read_rows(fh, f"head{l}", h["experts"], d, ln) for l in range(h["moe_layers"])])
        if fh.readline():
            raise TraceParseError("trailing data after parameter rows", line=ln[0] + 1)
    return SruParams(layers=layers, heads=heads)


def load_sru_params_device(path, device=None) -> "DeviceSru":
    """load_sru_params + the device layout the kernels use (bf16 W_cat, fp32 b_cat, heads)."""
    return _device_sru(load_sru_params(path), device or require_device())
