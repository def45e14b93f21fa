"""Device adapters of the file formats: parameters and batches loaded from the
reference-written files drive the CUDA path, checked against the CPU oracle."""

from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import moesim_oracle as O  # noqa: E402
from paper_2605_11537_b200.predictor import load_sru_params, sru_forward  # noqa: E402
from paper_2605_11537_b200.router_oracle import load_params, load_params_device, moe_forward, route_device  # noqa: E402
from paper_2605_11537_b200.workload import batch_to_device, load_trace_device, read_trace  # noqa: E402

IO = Path(__file__).resolve().parent / "golden" / "io"


def test_device_adapters_against_oracle():
    tr, dev_batches = load_trace_device(IO / "trace.txt")
    mp = load_params(IO / "moe_params.txt")
    dm = load_params_device(IO / "moe_params.txt")
    for b, (x, r) in zip(tr.batches, dev_batches):
        assert np.array_equal(r.cpu().numpy(), b.oracle_routing)
        for l in range(mp.num_layers):  # routing of the file's embeddings with the file's router, exact
            got = route_device(batch_to_device(b, d_pad=dm.layers[l].dp)[0], dm.layers[l]).cpu().numpy()
            ref = np.array([O.route_top1(mp.router_weights[l], b.embeddings[t]) for t in range(b.embeddings.shape[0])])
            assert np.array_equal(got, ref), l
        y = moe_forward(b, mp)
        yref, _ = O.moe_forward(b.embeddings, mp.router_weights, mp.expert_u, mp.expert_v)
        assert np.abs(y - yref).max() / np.abs(yref).max() <= 1e-2
    sp = load_sru_params(IO / "sru_params.txt")
    emb = read_trace(IO / "trace.txt").batches[0].embeddings
    h = sru_forward(emb, sp)
    href = O.sru_forward(emb.astype(np.float64), [(l.w, l.w_f, l.w_r, l.b_f, l.b_r) for l in sp.layers])
    assert np.abs(h - href).max() / np.abs(href).max() <= 1e-2
