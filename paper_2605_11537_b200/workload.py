"""Trace and parameter files -- drop-in for the reference's file formats
(SURVEY.md §8(f) rank 3), plus adapters that put their contents on the device.

Formats (line-delimited text, byte-compatible with the reference writers):
  * ``moesim-trace v1``      header ``layers= experts= d_model= batch_size= num_batches=
    skew= seed= hot_experts=``, then one line per token ``batch position e_0..e_{L-1}
    x_0..x_{d-1}`` (float32, 9 significant digits) in (batch, position) order
    (reference src/workload.py:315-436);
  * ``moesim-sru-params v1`` rows ``w{i} wf{i} wr{i} bf{i} br{i}`` per SRU layer, then
    ``head{l}`` rows (float64, 17 significant digits) (src/predictor.py:400-468);
  * ``moesim-moe-params v1`` rows ``router``, ``expert_u``, ``expert_v`` (float32, 9
    digits) (src/router_oracle.py:184-251) -- in router_oracle.save_params/load_params.
Errors follow the reference: ``TraceParseError(line=)`` for malformed files,
``ValidationError`` for out-of-range expert indices.

The parsers are host code (text in, numpy out); ``batch_to_device`` /
``load_*_device`` hand the arrays to the kernels in their device layouts.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .errors import TraceParseError, ValidationError
from .predictor import check_finite

TRACE_FORMAT_VERSION = "1"


def _positive(name: str, value: int, minimum: int = 1) -> None:
    if int(value) < minimum:
        raise ValidationError(f"{name} must be >= {minimum}, got {value}")


@dataclass(frozen=True)
class ModelShape:
    """Dimensions of the MoE model a trace is generated for (src/workload.py:28-41)."""

    num_layers: int
    experts_per_layer: int
    d_model: int
    batch_size: int = 64

    def __post_init__(self):
        _positive("num_layers", self.num_layers)
        _positive("experts_per_layer", self.experts_per_layer, 2)
        _positive("d_model", self.d_model, 2)
        _positive("batch_size", self.batch_size)


@dataclass
class Batch:
    """Embeddings (T, d) float32 plus per-layer oracle experts (L, T) int64 (src/workload.py:44-80)."""

    index: int
    embeddings: np.ndarray
    oracle_routing: np.ndarray

    def validate(self, shape: ModelShape) -> None:
        if self.embeddings.shape != (shape.batch_size, shape.d_model):
            raise ValidationError(f"batch {self.index}: embeddings shape {self.embeddings.shape} does not match "
                                  f"{(shape.batch_size, shape.d_model)}")
        if self.oracle_routing.shape != (shape.num_layers, shape.batch_size):
            raise ValidationError(f"batch {self.index}: oracle_routing shape {self.oracle_routing.shape} does not "
                                  f"match {(shape.num_layers, shape.batch_size)}")
        check_finite(f"batch {self.index} embeddings", self.embeddings)
        if self.oracle_routing.min() < 0 or self.oracle_routing.max() >= shape.experts_per_layer:
            raise ValidationError(f"batch {self.index}: expert index outside [0, {shape.experts_per_layer})")

    def __eq__(self, other):
        if not isinstance(other, Batch):
            return NotImplemented
        return (self.index == other.index and self.embeddings.dtype == other.embeddings.dtype
                and self.embeddings.shape == other.embeddings.shape
                and self.embeddings.tobytes() == other.embeddings.tobytes()
                and np.array_equal(self.oracle_routing, other.oracle_routing))


@dataclass
class RoutingTrace:
    """Ordered batches plus the generator settings of the file header (src/workload.py:83-101)."""

    shape: ModelShape
    batches: list
    skew: float = 0.0
    seed: int = 0
    hot_experts: int = 0

    def __post_init__(self):
        if not self.batches:
            raise ValidationError("a trace needs at least one batch")
        for b in self.batches:
            b.validate(self.shape)

    @property
    def num_batches(self) -> int:
        return len(self.batches)


def fmt_f32(v) -> str:
    """9 significant digits: an exact float32 round trip."""
    return f"{float(v):.9g}"


def fmt_f64(v) -> str:
    """17 significant digits: an exact float64 round trip."""
    return f"{float(v):.17g}"


def write_trace(trace: RoutingTrace, path) -> None:
    s = trace.shape
    head = (f"moesim-trace v{TRACE_FORMAT_VERSION} layers={s.num_layers} experts={s.experts_per_layer} "
            f"d_model={s.d_model} batch_size={s.batch_size} num_batches={trace.num_batches} "
            f"skew={trace.skew!r} seed={trace.seed} hot_experts={trace.hot_experts}")
    out = [head]
    for b in trace.batches:
        routing = np.asarray(b.oracle_routing)
        for t in range(s.batch_size):
            out.append(f"{b.index} {t} " + " ".join(str(int(e)) for e in routing[:, t]) + " "
                       + " ".join(fmt_f32(v) for v in b.embeddings[t]))
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(out) + "\n")


def _header_fields(line: str, magic: str, lineno: int = 1) -> dict:
    parts = line.split()
    if len(parts) < 2 or parts[0] != magic or parts[1] != f"v{TRACE_FORMAT_VERSION}":
        raise TraceParseError(f"not a {magic} v{TRACE_FORMAT_VERSION} header", line=lineno)
    fields = {}
    for p in parts[2:]:
        k, sep, v = p.partition("=")
        if not sep:
            raise TraceParseError(f"malformed header field {p!r}", line=lineno)
        fields[k] = v
    return fields


def read_trace(path) -> RoutingTrace:
    with open(path, encoding="utf-8") as fh:
        header = fh.readline()
        if not header.strip():
            raise TraceParseError("empty file", line=1)
        f = _header_fields(header.strip(), "moesim-trace")
        need = ("layers", "experts", "d_model", "batch_size", "num_batches", "skew", "seed")
        missing = [k for k in need if k not in f]
        if missing:
            raise TraceParseError(f"header missing fields: {', '.join(missing)}", line=1)
        try:
            shape = ModelShape(int(f["layers"]), int(f["experts"]), int(f["d_model"]), int(f["batch_size"]))
            nb, skew, seed = int(f["num_batches"]), float(f["skew"]), int(f["seed"])
            hot = int(f.get("hot_experts", "0"))
        except ValueError as exc:
            raise TraceParseError(f"bad header value: {exc}", line=1) from exc
        L, T, d = shape.num_layers, shape.batch_size, shape.d_model
        emb = np.zeros((nb, T, d), dtype=np.float32)
        routing = np.zeros((nb, L, T), dtype=np.int64)
        total = nb * T
        lineno, n = 1, 0
        for raw in fh:
            lineno += 1
            tok = raw.split()
            if not tok:
                raise TraceParseError("blank token line", line=lineno)
            if len(tok) != 2 + L + d:
                raise TraceParseError(f"expected {2 + L + d} fields, found {len(tok)}", line=lineno)
            if n >= total:
                raise TraceParseError("more token lines than the header declares", line=lineno)
            try:
                b, t = int(tok[0]), int(tok[1])
                ex = np.array([int(v) for v in tok[2:2 + L]], dtype=np.int64)
                vals = np.array([float(v) for v in tok[2 + L:]], dtype=np.float32)
            except ValueError as exc:
                raise TraceParseError(f"bad field: {exc}", line=lineno) from exc
            eb, et = divmod(n, T)
            if (b, t) != (eb, et):
                raise TraceParseError(f"token out of order: expected batch={eb} position={et}, found batch={b} "
                                      f"position={t}", line=lineno)
            if (ex < 0).any() or (ex >= shape.experts_per_layer).any():
                raise ValidationError(f"line {lineno}: expert index outside [0, {shape.experts_per_layer})")
            routing[b, :, t] = ex
            emb[b, t] = vals
            n += 1
        if n != total:
            raise TraceParseError(f"truncated file: expected {total} token lines, found {n}", line=lineno + 1)
    return RoutingTrace(shape, [Batch(b, emb[b], routing[b]) for b in range(nb)], skew=skew, seed=seed,
                        hot_experts=hot)


def read_rows(fh, tag: str, rows: int, width: int, lineno: list, dtype=np.float64) -> np.ndarray:
    """``rows`` lines ``tag v_0 .. v_{width-1}`` (shared by the parameter formats)."""
    out = np.zeros((rows, width), dtype=dtype)
    for i in range(rows):
        lineno[0] += 1
        raw = fh.readline()
        if not raw:
            raise TraceParseError(f"truncated file while reading {tag}", line=lineno[0])
        tok = raw.split()
        if len(tok) != width + 1 or tok[0] != tag:
            raise TraceParseError(f"expected a {tag} row of {width} values", line=lineno[0])
        try:
            out[i] = [float(v) for v in tok[1:]]
        except ValueError as exc:
            raise TraceParseError(f"bad float: {exc}", line=lineno[0]) from exc
    return out


def parse_param_header(line: str, magic: str, keys) -> dict:
    parts = line.split()
    if len(parts) < 2 or parts[0] != magic:
        raise TraceParseError(f"not a {magic} file", line=1)
    try:
        fields = dict(p.split("=", 1) for p in parts[2:])
        return {k: int(fields[k]) for k in keys}
    except (ValueError, KeyError) as exc:
        raise TraceParseError(f"bad header: {exc}", line=1) from exc


def batch_to_device(batch, device=None, d_pad: int | None = None):
    """(embeddings (T, d_pad) fp32, oracle routing (L, T) int32) as device tensors for the
    kernels (zero-padded columns when d_pad > d)."""
    from ._dev import require_device

    dev = device or require_device()
    emb = np.asarray(getattr(batch, "embeddings", batch), dtype=np.float32)
    T, d = emb.shape
    x = torch.zeros(T, d_pad or d, dtype=torch.float32, device=dev)
    x[:, :d] = torch.from_numpy(np.ascontiguousarray(emb)).to(dev)
    routing = getattr(batch, "oracle_routing", None)
    r = torch.from_numpy(np.asarray(routing, dtype=np.int32)).to(dev) if routing is not None else None
    return x, r


def load_trace_device(path, device=None):
    """read_trace + batch_to_device for every batch: (trace, [(x, routing), ...])."""
    tr = read_trace(path)
    return tr, [batch_to_device(b, device) for b in tr.batches]
