"""Pin the CPU oracle (oracle/moesim_oracle.py) to vectors produced by the
reference package itself (tests/golden/make_golden.py). CPU only."""

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import moesim_oracle as O

G = Path(__file__).resolve().parent / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def meta():
    return json.loads((G / "meta.json").read_text())


def test_cap_replicas_closed_form_and_walk():
    cases = json.loads((G / "planner.json").read_text())
    assert len(cases) > 3000
    for c in cases:
        dem = {int(e): int(n) for e, n in c["demand"]}
        exp = None if c["caps"] is None else {int(e): int(n) for e, n in c["caps"]}
        for fn in (O.cap_replicas, O.cap_replicas_walk):
            if exp is None:
                with pytest.raises(O.Infeasible):
                    fn(dem, c["capacity"])
            else:
                assert fn(dem, c["capacity"]) == exp


def _plan_dense(plan_layer, E):
    caps = np.zeros(E, dtype=np.int64)
    for e, n in plan_layer:
        caps[e] = n
    return caps


def test_apply_layer_closed_form_and_walk():
    cases = json.loads((G / "placement.json").read_text())
    for case in cases:
        L, E, C = case["L"], case["E"], case["capacity"]
        res = np.zeros((L, E), dtype=np.int64)
        resident = [dict() for _ in range(L)]
        for b in case["batches"]:
            a = np.array(b["assignment"])
            ev_all = []
            fb_all = []
            for l in range(L):
                caps = _plan_dense(b["plan"][l], E)
                plan_d = {int(e): int(n) for e, n in b["plan"][l]}
                tts_w, ev_w, fb_w = O.apply_layer_walk(resident[l], a[l], plan_d, C, b["plan_capacity"])
                tts, res_new, offl, ek, eo, fb = O.apply_layer(res[l], a[l], caps, C, b["plan_capacity"])
                assert tts.tolist() == b["token_to_slot"][l] == tts_w.tolist()
                assert fb == fb_w
                res[l] = res_new
                slots = sorted((e, o) for e in range(E) for o in range(res[l][e]))
                assert [list(s) for s in slots] == b["slots"][l]
                ev_all += [[k, l, e, o] for k, e, o in ev_w]
                if fb:
                    fb_all.append(l)
                # closed-form event counts
                assert int(offl.sum()) == sum(1 for k, _, _ in ev_w if k == O.OFFLOAD)
                assert int((ek > 0).sum()) == sum(1 for k, _, _ in ev_w if k != O.OFFLOAD)
            assert ev_all == b["events"]
            assert fb_all == b["fallback_layers"]


def test_execution_map_closed_form_and_walk():
    cases = json.loads((G / "exec.json").read_text())
    for case in cases:
        L, E, C = case["L"], case["E"], case["capacity"]
        res = np.zeros((L, E), dtype=np.int64)
        resident = [dict() for _ in range(L)]
        for b in case["batches"]:
            pred = np.array(b["predicted"])
            true = np.array(b["oracle"])
            plan = O.plan_all_layers(pred, C, on_infeasible="fallback")
            for l in range(L):
                caps = np.zeros(E, dtype=np.int64)
                for e, n in plan[l].items():
                    caps[e] = n
                tts, res[l], *_ = O.apply_layer(res[l], pred[l], caps, C, C)
                O.apply_layer_walk(resident[l], pred[l], dict(plan[l]), C, C)
                assert tts.tolist() == b["placement_token_to_slot"][l]
            for l in range(L):
                tts, cnt, corr = O.exec_map(res[l], true[l])
                tts_w, _, slots = O.exec_map_walk(resident[l], true[l])
                assert tts.tolist() == tts_w.tolist() == b["exec_token_to_slot"][l]
                res[l] = cnt
                assert [list(s) for s in slots] == b["exec_slots"][l]


def _sru_layers(z, key, S):
    return [tuple(z[f"{key}_l{s}_{nm}"] for nm in ("w", "w_f", "w_r", "b_f", "b_r")) for s in range(S)]


def test_sru_forward_and_predict(meta):
    z = np.load(G / "sru.npz")
    for m in meta["sru"]:
        k = m["key"]
        if "init_seed" in m:
            layers, heads = O.init_sru_params(m["L"], m["E"], m["d"], m["S"], m["init_seed"])
            flat = np.concatenate([np.concatenate([a.ravel() for a in lay]) for lay in layers] + [heads.ravel()])
            assert sha(flat) == m["weights_sha"]
        else:
            layers, heads = _sru_layers(z, k, m["S"]), z[f"{k}_heads"]
        x = z[f"{k}_x"]
        h = O.sru_forward(x, layers)
        np.testing.assert_allclose(h, z[f"{k}_h"], rtol=1e-10, atol=1e-12)
        if m["T"] <= 64:
            np.testing.assert_allclose(O.sru_forward_walk(x, layers), z[f"{k}_h"], rtol=1e-12, atol=1e-14)
        assign, _ = O.predict_assignment(x, layers, heads)
        assert (assign == z[f"{k}_assign"]).all()


def test_sparsemax_known_answers():
    assert np.allclose(O.sparsemax(np.array([0.0, 0.0])), [0.5, 0.5])
    assert np.allclose(O.sparsemax(np.array([10.0, 0.0])), [1.0, 0.0])
    assert np.allclose(O.sparsemax(np.array([0.5, 0.1, 0.05])), [0.6167, 0.2167, 0.1667], atol=1e-4)
    rng = np.random.default_rng(0)
    z = rng.normal(size=(500, 9)) * rng.uniform(0.1, 5.0, size=(500, 1))
    rows = O.sparsemax_rows(z)
    for i in range(500):
        assert np.allclose(rows[i], O.sparsemax(z[i]), atol=1e-12)
    # F3: argmax(sparsemax(z)) == argmax(z), including forced ties
    z[:50, 3] = z[:50].max(axis=1)
    assert (np.argmax(O.sparsemax_rows(z), axis=1) == np.argmax(z, axis=1)).all()


def test_moe_forward_random_configs(meta):
    z = np.load(G / "moe.npz")
    for m in meta["moe"]:
        k = m["key"]
        emb, router, u, v = z[f"{k}_emb"], z[f"{k}_router"], z[f"{k}_u"], z[f"{k}_v"]
        out_w, route_w = O.moe_forward_walk(emb, router, u, v)
        assert out_w.tobytes() == z[f"{k}_out"].tobytes()  # the walk is bit-identical to the reference
        assert (route_w == z[f"{k}_route"]).all()
        out_b, route_b = O.moe_forward(emb, router, u, v)
        assert (route_b == z[f"{k}_route"]).all()
        np.testing.assert_allclose(out_b, z[f"{k}_out"], rtol=1e-5, atol=1e-5)


def test_workload_restatement_is_bit_exact(meta):
    for pin in meta["workload"]:
        if "hot" in pin:
            continue
        L, E, d, T, nb, skew, seed = pin["args"]
        tr = O.generate_trace(L, E, d, T, nb, skew, seed)
        assert [sha(e) for e, _ in tr] == pin["emb"]
        assert [sha(r) for _, r in tr] == pin["route"]
        router, u, v = O.oracle_params_for_trace(L, E, d, seed, d_ff=2 * d)
        assert sha(router) == pin["router"] and sha(u) == pin["u"] and sha(v) == pin["v"]


def test_config1_end_to_end(meta):
    """BASELINE config 1 (8 experts, d=128, d_ff=512, 256 tokens): oracle == reference."""
    z = np.load(G / "moe.npz")
    c = meta["cfg1"]
    tr = O.generate_trace(1, 8, 128, 256, 2, c["skew"], c["seed"])
    router, u, v = O.oracle_params_for_trace(1, 8, 128, c["seed"], d_ff=c["d_ff"])
    assert sha(router) == c["params_sha"]["router"] and sha(u) == c["params_sha"]["u"]
    for b, (emb, route) in enumerate(tr):
        assert sha(emb) == c["batches"][b]["emb_sha"]
        out, chosen = O.moe_forward(emb, router, u, v)
        assert (chosen == z[f"cfg1_b{b}_route"]).all()
        np.testing.assert_allclose(out, z[f"cfg1_b{b}_out"], rtol=1e-5, atol=1e-5)
    layers, heads = O.init_sru_params(1, 8, 128, 10, c["sru_seed"])
    assert sha(heads) == c["sru_heads_sha"]
    assign, hidden = O.predict_assignment(tr[0][0], layers, heads)
    np.testing.assert_allclose(hidden, z["cfg1_pred_hidden"], rtol=1e-10, atol=1e-12)
    assert (assign == z["cfg1_pred_assign"]).all()


def test_training_oracle_matches_reference_bitwise():
    """oracle/training_oracle.py == the reference's loss_and_grads / train_predictor
    (tests/golden/train.npz), bit for bit."""
    from oracle import training_oracle as TO
    from oracle.moesim_oracle import init_sru_params

    z = np.load(G / "train.npz")
    for k in range(3):
        S, T, d, L, E, nl, seed = (int(v) for v in z[f"g{k}_meta"])
        layers, heads = init_sru_params(L, E, d, nl, seed)
        loss, lg, hg = TO.loss_and_grads(layers, heads, z[f"g{k}_x"], z[f"g{k}_y"])
        assert loss == float(z[f"g{k}_loss"])
        assert np.array_equal(hg, z[f"g{k}_heads"])
        for i in range(nl):
            for j, n in enumerate(("w", "w_f", "w_r", "b_f", "b_r")):
                assert np.array_equal(lg[i][j], z[f"g{k}_{i}_{n}"])
    layers, heads, curve = TO.train_predictor(z["t_emb"], z["t_lab"], 2, 4, 16, 4, 0.01, 3, 2, 5)
    assert np.array_equal(np.array(curve), z["t_curve"])
    assert np.array_equal(heads, z["t_heads"])
