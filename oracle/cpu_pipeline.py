"""Timed CPU run of the reference hot path on a bounded token sample -- TEST /
BASELINE INFRASTRUCTURE (bench.py's ``cpu_baseline`` and ``--impl reference``).

The chain is the reference's BatchRunner._run_predicted (src/simulator.py:181-208)
plus the MoE forward (src/router_oracle.py:119-135), restated in numpy by
``oracle/moesim_oracle.py`` (pinned to the reference's golden vectors):

  predict_batch (float64 SRU, S layers, head argmax)      src/predictor.py:212-223
  plan (cap_replicas per layer, fallback {})              src/simulator.py:135-146
  apply_layer per layer (closed form F5)                  src/placement.py:109-165
  per MoE layer: route_top1 (float64), execution map (F6), expert FFN (float32 BLAS,
  batched per expert) + residual add                     src/router_oracle.py:90-134

Bounded sample: ``tokens`` tokens of a Switch-base batch. All L MoE layers are
run; to bound host memory they share one layer's expert weights (the FLOP and
byte cost per layer is identical; weights never fit in CPU caches either way),
each layer with its own router. Timing uses every host thread (numpy/OpenBLAS).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import moesim_oracle as O


def host_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class CpuSample:
    def __init__(self, tokens=2048, L=12, E=128, d=768, F=3072, S=10, capacity=296, demand_unit=128, seed=0,
                 skew=1.2, constructed_predictor=True):
        rng = np.random.default_rng(seed)
        self.L, self.E, self.d, self.F, self.S = L, E, d, F, S
        self.C, self.unit = capacity, demand_unit
        k, cent, pop, perms = O.build_geometry(L, E, d, rng)
        probs = O.zipf_probabilities(E, skew, pop)
        e0 = rng.choice(E, size=tokens, p=probs)
        self.emb = O._margin_embeddings(k, cent, e0, rng, 0.1)
        self.router = np.empty((L, E, d), dtype=np.float32)
        for layer in range(L):
            self.router[layer, perms[layer]] = cent
        self.u = (rng.standard_normal((E, F, d), dtype=np.float32) / np.float32(np.sqrt(d)))
        self.v = (rng.standard_normal((E, d, F), dtype=np.float32) / np.float32(np.sqrt(F)))
        self.v[:, :k, :] = 0.0
        layers, heads = O.init_sru_params(L, E, d, S, seed + 1)
        if constructed_predictor:  # same construction as the GPU engine: highway-open, heads = router rows
            layers = [(w, wf, wr, bf, br - 8.0) for (w, wf, wr, bf, br) in layers]
            heads = self.router.astype(np.float64)
        self.sru_layers, self.heads = layers, heads

    def run(self):
        """One timed pass over the sample; returns (seconds, breakdown dict)."""
        L, E = self.L, self.E
        t0 = time.perf_counter()
        assign, _ = O.predict_assignment(self.emb, self.sru_layers, self.heads)
        t1 = time.perf_counter()
        res = np.zeros((L, E), dtype=np.int64)
        for l in range(L):
            dem = np.bincount(assign[l], minlength=E)
            dd = {int(e): int(-(-n // self.unit)) for e, n in enumerate(dem) if n}
            try:
                caps_d = O.cap_replicas(dd, self.C)
            except O.Infeasible:
                caps_d = {}
            caps = np.zeros(E, dtype=np.int64)
            for e, c in caps_d.items():
                caps[e] = c
            _, res[l], *_ = O.apply_layer(res[l], assign[l], caps, self.C, self.C)
        t2 = time.perf_counter()
        stream = self.emb.copy()
        for l in range(L):
            e_t = np.argmax(stream.astype(np.float64) @ self.router[l].astype(np.float64).T, axis=1)
            _, res[l], _ = O.exec_map(res[l], e_t)
            for e in np.unique(e_t):
                idx = np.nonzero(e_t == e)[0]
                xs = stream[idx]
                stream[idx] = xs + np.maximum(xs @ self.u[e].T, 0.0) @ self.v[e].T
        t3 = time.perf_counter()
        return t3 - t0, {"predict_s": t1 - t0, "plan_place_s": t2 - t1, "forward_s": t3 - t2}
