"""SRU predictor training on the GPU -- drop-in for the training half of
``moesim.predictor`` (reference src/predictor.py:238-379).

Same functions, signatures, results and errors: ``loss_and_grads(params, embeddings,
labels) -> (loss, SruParams grads)``, ``train_predictor(trace, epochs, learning_rate,
seed, num_sru_layers, sequences_per_step) -> TrainingResult``, ``TrainingError`` naming
the epoch on divergence, ``ConfigurationError`` on bad arguments. Float64 like the
reference. The recurrences (forward with caches, back-propagation through time of the
cell state), the softmax cross-entropy, the reductions and the SGD update run in
libmoempmc (csrc/train.cu, no FMA contraction so the cell updates round like the
reference's numpy expressions); the dense products are the library's own float64 GEMM
(``mp_dgemm``, csrc/dgemm.cu).
Parameters stay on the device for the whole run; the loss of every step is read back
(the reference checks it for finiteness per step, src/predictor.py:364-367).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._dev import ptr, require_device, stream_ptr
from .errors import ConfigurationError, TrainingError
from .predictor import DEFAULT_SRU_LAYERS, SruLayerParams, SruParams, init_params

_NAMES = ("w", "w_f", "w_r", "b_f", "b_r")


@dataclass
class TrainingResult:
    params: SruParams
    loss_curve: list


class _DevParams:
    """SruParams as float64 device tensors."""

    def __init__(self, params: SruParams, dev):
        self.layers = [{k: torch.from_numpy(np.ascontiguousarray(getattr(l, k), dtype=np.float64)).to(dev)
                        for k in _NAMES} for l in params.layers]
        self.heads = torch.from_numpy(np.ascontiguousarray(params.heads, dtype=np.float64)).to(dev)

    def tensors(self):
        for l in self.layers:
            for k in _NAMES:
                yield l[k]
        yield self.heads

    def to_host(self) -> SruParams:
        return SruParams(layers=[SruLayerParams(*(l[k].cpu().numpy() for k in _NAMES)) for l in self.layers],
                         heads=self.heads.cpu().numpy())


def _axpy(y: torch.Tensor, x: torch.Tensor, alpha: float, sp: int) -> None:
    _lib.call("mp_train_axpy", ptr(y), ptr(x), y.numel(), float(alpha), sp)


def _mm(a: torch.Tensor, b: torch.Tensor, ta: bool = False, tb: bool = False, out: torch.Tensor | None = None,
        accumulate: bool = False) -> torch.Tensor:
    """op(a) @ op(b) in float64 through mp_dgemm (op = transpose when ta / tb); with
    ``accumulate`` the product is added to ``out``."""
    a, b = a.contiguous(), b.contiguous()
    M, K = (a.shape[1], a.shape[0]) if ta else a.shape
    N = b.shape[0] if tb else b.shape[1]
    if out is None:
        out = torch.empty(M, N, dtype=torch.float64, device=a.device)
    _lib.call("mp_dgemm", int(ta), int(tb), M, N, K, ptr(a), a.shape[1], ptr(b), b.shape[1],
              1.0 if accumulate else 0.0, ptr(out), N, stream_ptr())
    return out


def _loss_and_grads_dev(p: _DevParams, x: torch.Tensor, labels: torch.Tensor):
    """x (S, T, d) float64, labels (S, L, T) int64 on the device -> (loss, grads as _DevParams-like)."""
    sp = stream_ptr()
    S, T, d = x.shape
    N = S * T
    L, E = p.heads.shape[0], p.heads.shape[1]
    f64 = dict(dtype=torch.float64, device=x.device)
    caches = []
    h = x
    for lay in p.layers:  # forward with caches (src/predictor.py:238-254)
        xf = h.reshape(N, d)
        u = _mm(xf, lay["w"], tb=True)
        fm = _mm(xf, lay["w_f"], tb=True)
        rm = _mm(xf, lay["w_r"], tb=True)
        f, r, c, g, hn = (torch.empty(S, T, d, **f64) for _ in range(5))
        _lib.call("mp_sru_train_fwd", ptr(u), ptr(fm), ptr(rm), ptr(lay["b_f"]), ptr(lay["b_r"]), ptr(h), S, T, d,
                  ptr(f), ptr(r), ptr(c), ptr(g), ptr(hn), sp)
        caches.append((h, u, f, r, c, g))
        h = hn
    hf = h.reshape(N, d)
    dh = torch.zeros(N, d, **f64)
    head_grads = torch.empty(L, E, d, **f64)
    dz = torch.empty(N, E, **f64)
    row_loss = torch.empty(N, **f64)
    lsum = torch.empty(L, **f64)
    for l in range(L):  # heads: softmax cross-entropy (src/predictor.py:310-326)
        z = _mm(hf, p.heads[l], tb=True)
        _lib.call("mp_train_ce", ptr(z), ptr(labels), S, T, L, l, E, ptr(dz), ptr(row_loss), sp)
        _lib.call("mp_train_sum", ptr(row_loss), N, ptr(lsum[l:l + 1]), sp)
        _mm(dz, hf, ta=True, out=head_grads[l])
        _mm(dz, p.heads[l], out=dh, accumulate=True)
    grads = []
    bsf, bsr = torch.empty(S, d, **f64), torch.empty(S, d, **f64)
    for lay, (xc, u, f, r, c, g) in zip(reversed(p.layers), reversed(caches)):  # BPTT (src/predictor.py:257-294)
        du, dfp, drp, dho = (torch.empty(S, T, d, **f64) for _ in range(4))
        _lib.call("mp_sru_train_bwd", ptr(dh), ptr(xc), ptr(u), ptr(f), ptr(r), ptr(c), ptr(g), S, T, d, ptr(du),
                  ptr(dfp), ptr(drp), ptr(dho), ptr(bsf), ptr(bsr), sp)
        xf = xc.reshape(N, d)
        gl = {"w": _mm(du.reshape(N, d), xf, ta=True), "w_f": _mm(dfp.reshape(N, d), xf, ta=True),
              "w_r": _mm(drp.reshape(N, d), xf, ta=True),
              "b_f": torch.empty(d, **f64), "b_r": torch.empty(d, **f64)}
        _lib.call("mp_train_colsum", ptr(bsf), S, d, ptr(gl["b_f"]), sp)
        _lib.call("mp_train_colsum", ptr(bsr), S, d, ptr(gl["b_r"]), sp)
        dho = dho.reshape(N, d)
        _mm(du.reshape(N, d), lay["w"], out=dho, accumulate=True)
        _mm(dfp.reshape(N, d), lay["w_f"], out=dho, accumulate=True)
        _mm(drp.reshape(N, d), lay["w_r"], out=dho, accumulate=True)
        dh = dho
        grads.append(gl)
    grads.reverse()
    loss = sum(float(v) / S for v in lsum.cpu().tolist())  # per layer: sum / num_sequences
    return loss, grads, head_grads


def _inputs(embeddings, labels, dev):
    x = torch.from_numpy(np.ascontiguousarray(embeddings, dtype=np.float64)).to(dev)
    y = torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int64)).to(dev)
    if x.ndim != 3 or y.ndim != 3 or y.shape[0] != x.shape[0] or y.shape[2] != x.shape[1]:
        raise ConfigurationError(f"embeddings {tuple(x.shape)} / labels {tuple(y.shape)} shape mismatch")
    return x, y


def loss_and_grads(params: SruParams, embeddings: np.ndarray, labels: np.ndarray):
    """Cross-entropy loss and gradients over a group of sequences (src/predictor.py:297-334)."""
    dev = require_device()
    x, y = _inputs(embeddings, labels, dev)
    p = _DevParams(params, dev)
    loss, grads, hg = _loss_and_grads_dev(p, x, y)
    layers = [SruLayerParams(*(g[k].cpu().numpy() for k in _NAMES)) for g in grads]
    return loss, SruParams(layers=layers, heads=hg.cpu().numpy())


def train_predictor(trace, epochs: int, learning_rate: float = 0.001, seed: int = 0,
                    num_sru_layers: int = DEFAULT_SRU_LAYERS, sequences_per_step: int = 32) -> TrainingResult:
    """Mini-batch SGD on a trace's oracle routing (src/predictor.py:343-379): each step consumes up
    to ``sequences_per_step`` batches in order; deterministic for a fixed seed."""
    if epochs < 0:
        raise ConfigurationError("epochs must be >= 0")
    if learning_rate <= 0:
        raise ConfigurationError("learning_rate must be > 0")
    shape = trace.shape
    params = init_params(shape.num_layers, shape.experts_per_layer, shape.d_model, num_sru_layers, seed)
    if epochs == 0:
        return TrainingResult(params=params, loss_curve=[])
    dev = require_device()
    x, y = _inputs(np.stack([b.embeddings for b in trace.batches]), np.stack([b.oracle_routing for b in trace.batches]),
                   dev)
    p = _DevParams(params, dev)
    n = x.shape[0]
    step = max(1, int(sequences_per_step))
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    sp = stream_ptr()
    losses = []
    for epoch in range(epochs):
        total = 0.0
        for a in range(0, n, step):
            b = min(a + step, n)
            loss, grads, hg = _loss_and_grads_dev(p, x[a:b].contiguous(), y[a:b].contiguous())
            if not np.isfinite(loss):
                raise TrainingError("training loss is not finite", epoch=epoch)
            total += loss * (b - a)
            for lay, g in zip(p.layers, grads):
                for k in _NAMES:
                    _axpy(lay[k], g[k], -learning_rate, sp)
            _axpy(p.heads, hg, -learning_rate, sp)
        for t in p.tensors():
            _lib.call("mp_train_nonfinite", ptr(t), t.numel(), ptr(flag), sp)
        if int(flag.item()):
            raise TrainingError("parameters diverged to non-finite values", epoch=epoch)
        losses.append(total / n)
    return TrainingResult(params=p.to_host(), loss_curve=losses)
