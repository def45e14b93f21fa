"""Parity of the CUDA path (through the reference-shaped Python API, i.e. the
C-ABI) with the reference: golden vectors produced by the reference package
(tests/golden/) and the pinned CPU oracle.

Bars (BASELINE.json north_star):
  * bit-exact: histograms, replica plans, placements (token maps, slots,
    transfer events, fallback flags), execution maps, true routing;
  * tolerance: SRU hidden states and FFN/combine outputs, max-norm relative
    error ||gpu - ref||_inf / ||ref||_inf <= 1e-2 (bf16 operands, fp32 acc);
    predicted-expert argmax flips are counted and reported.
"""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import moesim_oracle as O  # noqa: E402
from paper_2605_11537_b200 import (  # noqa: E402
    ConfigurationError,
    InfeasibleCapacityError,
    NumericError,
    PlacementError,
)
from paper_2605_11537_b200.placement import DeviceState, apply_batch, apply_layer, execution_map  # noqa: E402
from paper_2605_11537_b200.planner import (  # noqa: E402
    ReplicaPlan,
    cap_replicas,
    demand_counts,
    plan_all_layers,
    plan_layers_with_fallback,
)
from paper_2605_11537_b200.predictor import (  # noqa: E402
    HashTable,
    SruLayerParams,
    SruParams,
    init_params,
    predict_batch,
    sparsemax,
    sru_cell,
    sru_forward,
)
from paper_2605_11537_b200.router_oracle import (  # noqa: E402
    LayerPlacement,
    Placement,
    ToyMoeParams,
    expert_forward,
    moe_forward,
    oracle_route_batch,
    route_top1,
)

G = Path(__file__).resolve().parent / "golden"
TOL = 1e-2


def maxnorm_rel(a, b):
    return float(np.abs(np.asarray(a, np.float64) - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module")
def meta():
    return json.loads((G / "meta.json").read_text())


# ------------------------------------------------------------------ planner (bit-exact)


def test_cap_replicas_golden():
    cases = json.loads((G / "planner.json").read_text())
    for c in cases:
        dem = {int(e): int(n) for e, n in c["demand"]}
        if c["caps"] is None:
            with pytest.raises(InfeasibleCapacityError):
                cap_replicas(dem, c["capacity"])
        else:
            assert cap_replicas(dem, c["capacity"]) == {int(e): int(n) for e, n in c["caps"]}


def test_planner_known_answers_and_errors():
    assert cap_replicas({0: 10, 1: 5, 2: 1}, 8) == {0: 4, 1: 3, 2: 1}
    assert cap_replicas({0: 100, 1: 2}, 10) == {0: 8, 1: 2}
    assert cap_replicas({0: 3, 1: 3}, 5) == {0: 3, 1: 2}
    assert cap_replicas({}, 4) == {}
    with pytest.raises(ConfigurationError):
        cap_replicas({0: 1}, 0)
    table = HashTable.from_assignment(0, np.array([[0, 0, 0, 0], [0, 1, 2, 3]]))
    with pytest.raises(InfeasibleCapacityError) as ei:
        plan_all_layers(table, capacity=3)
    assert ei.value.layer == 1
    assert demand_counts(HashTable.from_assignment(0, np.array([[3, 1, 4, 2]])), 0) == {1: 1, 2: 1, 3: 1, 4: 1}
    with pytest.raises(ConfigurationError):
        demand_counts(table, 3)


def test_plan_all_layers_matches_oracle(rng):
    for _ in range(60):
        L, T, E = int(rng.integers(1, 5)), int(rng.integers(1, 3000)), int(rng.integers(2, 300))
        w = 1.0 / (rng.permutation(E) + 1.0) ** rng.uniform(0, 2)
        a = rng.choice(E, size=(L, T), p=w / w.sum())
        table = HashTable.from_assignment(0, a)
        assert table.replica_counts == O.histograms(a)
        distinct = max(len(set(r.tolist())) for r in a)
        C = int(rng.integers(distinct, 4 * distinct + 8))
        assert plan_all_layers(table, C).layers == O.plan_all_layers(a, C)


# ------------------------------------------------------------------ placement / execution (bit-exact)


def test_apply_batch_golden_sequences():
    cases = json.loads((G / "placement.json").read_text())
    for case in cases:
        state = DeviceState(case["L"], case["capacity"])
        for bi, b in enumerate(case["batches"]):
            table = HashTable.from_assignment(bi, np.array(b["assignment"]))
            plan = ReplicaPlan(b["plan_capacity"], [{int(e): int(n) for e, n in lay} for lay in b["plan"]])
            _, placement, log = apply_batch(state, table, plan)
            for l, lp in enumerate(placement.layers):
                assert lp.token_to_slot.tolist() == b["token_to_slot"][l]
                assert [list(s) for s in lp.slots] == b["slots"][l]
            assert [[e.kind, e.layer, e.expert, e.ordinal] for e in log.events] == b["events"]
            assert log.fallback_layers == b["fallback_layers"]


def test_apply_layer_hand_traces():
    # reference placement KATs (pkg/tests/test_placement.py:14-79)
    t = HashTable.from_assignment(0, np.array([[0] * 32 + [1] * 32]))
    st = DeviceState(1, 64)
    _, tts, log = apply_layer(st, t, ReplicaPlan(64, [{0: 32, 1: 32}]), 0)
    assert log.count("load") == 2 and log.count("replicate") == 62 and len(set(tts.tolist())) == 64
    st = DeviceState(1, 2)
    _, tts, _ = apply_layer(st, HashTable.from_assignment(0, np.array([[0] * 5])), ReplicaPlan(2, [{0: 2}]), 0)
    assert tts.tolist() == [0, 1, 0, 1, 0] and st.slots(0) == [(0, 0), (0, 1)]
    st = DeviceState(1, 8)
    apply_layer(st, HashTable.from_assignment(0, np.array([[0] * 5])), ReplicaPlan(8, [{0: 5}]), 0)
    _, _, log = apply_layer(st, HashTable.from_assignment(0, np.array([[0, 0]])), ReplicaPlan(8, [{0: 2}]), 0)
    assert [e.ordinal for e in log.events if e.kind == "offload"] == [4, 3, 2]
    st = DeviceState(1, 2)
    _, tts, log = apply_layer(st, HashTable.from_assignment(0, np.array([[0, 0, 1, 1, 2]])), ReplicaPlan(2, [{}]), 0)
    assert log.fallback_layers == [0] and {e for e, _ in st.slots(0)} == {0, 1, 2}
    with pytest.raises(ConfigurationError):
        apply_batch(DeviceState(2, 4), HashTable.from_assignment(0, np.array([[0]])), ReplicaPlan(4, [{0: 1}]))


def test_execution_map_golden():
    cases = json.loads((G / "exec.json").read_text())
    for case in cases:
        state = DeviceState(case["L"], case["capacity"])
        for bi, b in enumerate(case["batches"]):
            table = HashTable.from_assignment(bi, np.array(b["predicted"]))
            plan = plan_layers_with_fallback(table, case["capacity"])
            _, placement, log = apply_batch(state, table, plan)
            assert [lp.token_to_slot.tolist() for lp in placement.layers] == b["placement_token_to_slot"]
            _, ex, xlog = execution_map(state, np.array(b["oracle"]))
            log.extend(xlog)
            assert [lp.token_to_slot.tolist() for lp in ex.layers] == b["exec_token_to_slot"]
            assert [[list(s) for s in lp.slots] for lp in ex.layers] == b["exec_slots"]
            assert [[e.kind, e.layer, e.expert, e.ordinal] for e in log.events] == b["events"]
            assert log.fallback_layers == b["fallback_layers"]


def test_placement_large_matches_closed_form(rng):
    """GPU-scale rows (16k tokens, 128 experts) vs the oracle's closed forms (F5, F6)."""
    L, T, E, C = 3, 16384, 128, 296
    state = DeviceState(L, C)
    res = np.zeros((L, E), dtype=np.int64)
    for b in range(3):
        w = 1.0 / (rng.permutation(E) + 1.0) ** 1.2
        a = rng.choice(E, size=(L, T), p=w / w.sum())
        table = HashTable.from_assignment(b, a)
        plan = plan_layers_with_fallback(table, C)
        _, placement, log = apply_batch(state, table, plan)
        for l in range(L):
            caps = np.zeros(E, dtype=np.int64)
            for e, n in plan.layers[l].items():
                caps[e] = n
            tts, res[l], offl, ek, eo, fb = O.apply_layer(res[l], a[l], caps, C, C)
            assert (placement.layers[l].token_to_slot == tts).all()
        true = rng.choice(E, size=(L, T))
        _, ex, _ = execution_map(state, true)
        for l in range(L):
            tts, res[l], _ = O.exec_map(res[l], true[l])
            assert (ex.layers[l].token_to_slot == tts).all()


# ------------------------------------------------------------------ predictor (tolerance + flips)


def _sru_params(z, m):
    if "init_seed" in m:
        return init_params(m["L"], m["E"], m["d"], num_sru_layers=m["S"], seed=m["init_seed"])
    k = m["key"]
    layers = [SruLayerParams(*(z[f"{k}_l{s}_{nm}"] for nm in ("w", "w_f", "w_r", "b_f", "b_r")))
              for s in range(m["S"])]
    return SruParams(layers=layers, heads=z[f"{k}_heads"])


def test_sru_forward_and_predict_golden(meta):
    z = np.load(G / "sru.npz")
    report = []
    for m in meta["sru"]:
        params = _sru_params(z, m)
        x = z[f"{m['key']}_x"]
        h = sru_forward(x, params)
        err = maxnorm_rel(h, z[f"{m['key']}_h"])
        assert err <= TOL, (m, err)
        table = predict_batch(x, params)
        flips = int((table.assignment != z[f"{m['key']}_assign"]).sum())
        report.append((m["key"], err, flips, table.assignment.size))
        assert flips <= max(2, 0.02 * table.assignment.size), report
    print("SRU parity (key, max-norm rel err, argmax flips, cells):", report)


def test_sru_known_answers(rng):
    z3 = np.zeros((3, 3))
    h, c = sru_cell(np.zeros(3), np.zeros(3), SruLayerParams(z3, z3, z3, np.zeros(3), np.zeros(3)))
    assert np.array_equal(h, np.zeros(3)) and np.array_equal(c, np.zeros(3))
    lay = SruLayerParams(*(rng.normal(size=(4, 4)) for _ in range(3)), np.full(4, 50.0), rng.normal(size=4))
    c_prev = rng.normal(size=4)
    _, c = sru_cell(rng.normal(size=4), c_prev, lay)
    assert np.allclose(c, c_prev, atol=1e-6)  # saturated forget gate keeps the state
    x = rng.normal(size=(4, 6))
    zero = SruLayerParams(np.zeros((6, 6)), np.zeros((6, 6)), np.zeros((6, 6)), np.zeros(6), np.zeros(6))
    assert np.allclose(sru_forward(x, SruParams([zero], np.zeros((1, 2, 6)))), 0.5 * x, rtol=1e-6)
    assert np.allclose(sru_forward(x, SruParams([zero, zero], np.zeros((1, 2, 6)))), 0.25 * x, rtol=1e-6)
    with pytest.raises(ConfigurationError):
        sru_forward(np.zeros((0, 4)), init_params(1, 2, 4, num_sru_layers=1))
    with pytest.raises(NumericError):
        sru_forward(np.array([[np.nan, 0, 0, 0]]), init_params(1, 2, 4, num_sru_layers=1))


def test_sparsemax_known_answers(rng):
    assert np.allclose(sparsemax(np.array([0.0, 0.0])), [0.5, 0.5])
    assert np.allclose(sparsemax(np.array([10.0, 0.0])), [1.0, 0.0])
    assert np.allclose(sparsemax(np.array([0.5, 0.1, 0.05])), [0.6167, 0.2167, 0.1667], atol=1e-4)
    for _ in range(100):
        zz = rng.normal(size=int(rng.integers(2, 40))) * rng.uniform(0.1, 5)
        assert np.allclose(sparsemax(zz), O.sparsemax(zz), atol=1e-12)
    with pytest.raises(ConfigurationError):
        sparsemax(np.zeros(0))


def test_predict_batch_histogram_consistency(rng):
    params = init_params(3, 16, 32, num_sru_layers=2, seed=3)
    table = predict_batch(rng.normal(size=(500, 32)), params)
    assert table.replica_counts == O.histograms(table.assignment)


# ------------------------------------------------------------------ MoE forward


def _expert_placement(route):
    """Placement whose slots are the experts themselves (one replica each) following ``route``."""
    L, T = route.shape
    layers = []
    for l in range(L):
        ex = sorted(set(route[l].tolist()))
        pos = {e: i for i, e in enumerate(ex)}
        layers.append(LayerPlacement(slots=[(e, 0) for e in ex], token_to_slot=np.array([pos[e] for e in route[l]])))
    return Placement(layers)


def test_routing_bit_exact_on_reference_streams(meta):
    """route_top1 on the GPU == the reference's float64 argmax, layer by layer, when fed the
    reference's own residual stream (the oracle walk is bit-identical to the reference)."""
    from paper_2605_11537_b200._dev import require_device
    from paper_2605_11537_b200.router_oracle import _device_moe, route_device
    import torch

    z = np.load(G / "moe.npz")
    dev = require_device()
    for m in meta["moe"]:
        k = m["key"]
        router, u, v = z[f"{k}_router"], z[f"{k}_u"], z[f"{k}_v"]
        dm = _device_moe(ToyMoeParams(router, u, v), dev)
        stream = z[f"{k}_emb"].astype(np.float32).copy()
        for l in range(m["L"]):
            x = torch.zeros(m["T"], dm.dp)
            x[:, : m["d"]] = torch.from_numpy(stream)
            got = route_device(x.to(dev), dm.layers[l]).cpu().numpy()
            exp = np.array([O.route_top1(router[l], stream[t]) for t in range(m["T"])])
            assert (got == exp).all(), (k, l)
            assert (exp == z[f"{k}_route"][l]).all() or l > 0
            for t in range(m["T"]):
                stream[t] = stream[t] + O.expert_forward(stream[t], u[l, exp[t]], v[l, exp[t]])


def test_forward_golden_given_reference_routing(meta):
    """FFN + combine within tolerance given identical routing decisions; dense-baseline routing
    flips (bf16 FFN drift at later layers, random weights have no routing margin) are counted."""
    z = np.load(G / "moe.npz")
    flips = cells = 0
    for m in meta["moe"]:
        k = m["key"]
        params = ToyMoeParams(z[f"{k}_router"], z[f"{k}_u"], z[f"{k}_v"])
        emb, ref_route, ref_out = z[f"{k}_emb"], z[f"{k}_route"], z[f"{k}_out"]
        out = moe_forward(emb, params, _expert_placement(ref_route))
        assert maxnorm_rel(out, ref_out) <= TOL, k
        route = oracle_route_batch(emb, params)
        assert (route[0] == ref_route[0]).all(), k  # first layer sees identical inputs
        flips += int((route != ref_route).sum())
        cells += route.size
        ok = (route == ref_route).all(axis=0)
        dense = moe_forward(emb, params)
        if ok.any():
            assert maxnorm_rel(dense[ok], ref_out[ok]) <= TOL, k
    print(f"dense-baseline routing flips vs reference: {flips}/{cells}")
    assert flips <= 0.02 * cells


def test_replication_transparency_bitwise(meta):
    """Replicated placement == dense baseline bit for bit on the GPU (test_acceptance.py:45-70 analogue)."""
    z = np.load(G / "moe.npz")
    rng = np.random.default_rng(9)
    for m in meta["moe"]:
        k = m["key"]
        params = ToyMoeParams(z[f"{k}_router"], z[f"{k}_u"], z[f"{k}_v"])
        emb = z[f"{k}_emb"]
        route = oracle_route_batch(emb, params)
        out = moe_forward(emb, params)
        table = HashTable.from_assignment(0, route)
        distinct = max(len(set(r.tolist())) for r in route)
        C = int(rng.integers(distinct, max(m["T"], distinct) + 4))
        state = DeviceState(m["L"], C)
        _, placement, _ = apply_batch(state, table, plan_all_layers(table, C))
        assert moe_forward(emb, params, placement).tobytes() == out.tobytes(), k


def test_config1_against_reference(meta):
    """BASELINE config 1: 8 experts, d=128, d_ff=512, 256 tokens, Zipf 1.2 -- full pipeline."""
    z = np.load(G / "moe.npz")
    c = meta["cfg1"]
    tr = O.generate_trace(1, 8, 128, 256, 2, c["skew"], c["seed"])
    router, u, v = O.oracle_params_for_trace(1, 8, 128, c["seed"], d_ff=c["d_ff"])
    params = ToyMoeParams(router, u, v)
    for b, (emb, _) in enumerate(tr):
        assert hashlib.sha256(emb.tobytes()).hexdigest() == c["batches"][b]["emb_sha"]
        assert (oracle_route_batch(emb, params) == z[f"cfg1_b{b}_route"]).all()
        assert maxnorm_rel(moe_forward(emb, params), z[f"cfg1_b{b}_out"]) <= TOL
    sru = init_params(1, 8, 128, num_sru_layers=10, seed=c["sru_seed"])
    assert maxnorm_rel(sru_forward(tr[0][0], sru), z["cfg1_pred_hidden"]) <= TOL
    flips = int((predict_batch(tr[0][0], sru).assignment != z["cfg1_pred_assign"]).sum())
    print(f"config 1 predictor argmax flips: {flips}/256")
    assert flips <= 8


def test_router_and_expert_known_answers(rng):
    router = np.zeros((1, 8, 4), dtype=np.float32)
    router[0, 2] = [1, 0, 0, 0]
    router[0, 5] = [1, 0, 0, 0]
    p = ToyMoeParams(router, np.zeros((1, 8, 4, 4), np.float32), np.zeros((1, 8, 4, 4), np.float32))
    assert route_top1(0, np.array([1.0, 0, 0, 0]), p) == 2  # tie -> lower index
    with pytest.raises(NumericError):
        route_top1(0, np.array([np.nan, 0, 0, 0]), p)
    with pytest.raises(ConfigurationError):
        route_top1(1, np.zeros(4), p)
    u, v = rng.normal(size=(5, 3)), rng.normal(size=(3, 5))
    assert np.array_equal(expert_forward(np.zeros(3), u, v), np.zeros(3))
    x = np.array([0.5, 1.5, 0.0])
    assert np.array_equal(expert_forward(x, np.eye(3), np.eye(3)), x)
    xx = rng.normal(size=3)
    assert maxnorm_rel(expert_forward(xx, u, v), v @ np.maximum(u @ xx, 0)) <= TOL
    with pytest.raises(ConfigurationError):
        expert_forward(np.zeros(3), rng.normal(size=(4, 2)), rng.normal(size=(3, 4)))


def test_placement_errors(rng):
    from paper_2605_11537_b200.router_oracle import random_params

    class Shape:
        num_layers, experts_per_layer, d_model = 1, 3, 4

    params = random_params(Shape, seed=1)
    bad = Placement(layers=[LayerPlacement(slots=[(0, 0)], token_to_slot=np.array([0, 5]))])
    with pytest.raises(PlacementError):
        moe_forward(rng.normal(size=(2, 4)).astype(np.float32), params, bad)
    with pytest.raises(ConfigurationError):
        moe_forward(rng.normal(size=(2, 4)).astype(np.float32), params, "warp-speed")
