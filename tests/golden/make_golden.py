"""Generate golden vectors by running the REFERENCE package (``moesim``).

Run in the build container (the reference is not on the GPU box):

    python tests/golden/make_golden.py [/root/reference/pkg/src]

Writes small JSON / NPZ fixtures next to this file. They pin both the CPU
oracle (oracle/moesim_oracle.py) and, through it or directly, the CUDA path.
Every case is drawn from the same distributions the reference's own tests use
(pkg/tests/test_planner.py:69-104, test_placement.py:102-122,
test_acceptance.py:45-70) plus the reference's known-answer tests.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = next((a for a in sys.argv[1:] if not a.startswith("--")), "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import moesim  # noqa: E402
from moesim import (  # noqa: E402
    DeviceState,
    HashTable,
    InfeasibleCapacityError,
    ModelShape,
    ReplicaPlan,
    apply_batch,
    cap_replicas,
    generate_hot_trace,
    generate_trace,
    moe_forward,
    oracle_params_for_trace,
    oracle_route_batch,
    plan_all_layers,
    predict_batch,
    sru_forward,
)
from moesim.predictor import SruLayerParams, SruParams, init_params  # noqa: E402
from moesim.router_oracle import random_params  # noqa: E402
from moesim.simulator import BatchRunner, CostModel, simulate_strategy  # noqa: E402

OUT = Path(__file__).resolve().parent


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def planner_cases():
    cases = []
    kats = [
        ({0: 32, 1: 32}, 64), ({e: 1 for e in range(6)}, 6), ({e: 1 for e in range(6)}, 100),
        ({0: 10, 1: 5, 2: 1}, 8), ({0: 100, 1: 2}, 10), ({0: 3, 1: 3}, 5), ({0: 2, 1: 2, 2: 2}, 2), ({}, 4),
    ]
    rng = np.random.default_rng(11)
    rand = []
    for _ in range(3000):
        ids = rng.choice(300, size=int(rng.integers(1, 20)), replace=False)
        dem = {int(e): int(rng.integers(1, 60)) for e in ids}
        lo = max(1, len(dem) - 2)
        cap = int(rng.integers(lo, sum(dem.values()) + 5))
        rand.append((dem, cap))
    # GPU-scale shaped demands (Zipf-like, E = 128 / 256)
    for E in (128, 256):
        for _ in range(50):
            w = 1.0 / (rng.permutation(E) + 1.0) ** rng.uniform(0.0, 2.0)
            cnt = np.bincount(rng.choice(E, size=int(rng.integers(1000, 20000)), p=w / w.sum()), minlength=E)
            dem = {int(e): int(c) for e, c in enumerate(cnt) if c > 0}
            cap = int(rng.integers(len(dem), 4 * E))
            rand.append((dem, cap))
    for dem, cap in kats + rand:
        try:
            caps = cap_replicas(dem, cap)
            cases.append({"demand": sorted(dem.items()), "capacity": cap, "caps": sorted(caps.items())})
        except InfeasibleCapacityError:
            cases.append({"demand": sorted(dem.items()), "capacity": cap, "caps": None})
    return cases


def _events(log):
    return [[e.kind, e.layer, e.expert, e.ordinal] for e in log.events]


def placement_cases():
    """Sequences of batches through plan_all_layers/apply_batch (test_placement.py:102-122 style),
    plus fallback cases where a layer's plan is {} (simulator.py:142-145) or a foreign plan."""
    rng = np.random.default_rng(22)
    out = []
    for trial in range(400):
        L = int(rng.integers(1, 4))
        T = int(rng.integers(1, 40))
        E = int(rng.integers(2, 10))
        C = int(rng.integers(max(1, E - 3), E + 30))
        skew = float(rng.uniform(0.0, 2.0))
        p = 1.0 / (np.arange(E) + 1.0) ** skew
        p = rng.permutation(p / p.sum())
        state = DeviceState(L, C)
        batches = []
        for b in range(4):
            a = rng.choice(E, size=(L, T), p=p)
            table = HashTable.from_assignment(b, a)
            layers = []
            for l in range(L):
                dem = moesim.demand_counts(table, l)
                try:
                    layers.append(cap_replicas(dem, C))
                except InfeasibleCapacityError:
                    layers.append({})
            if trial % 7 == 0 and b == 2:  # foreign plan: caps for other experts / over capacity
                layers = [{int(e): int(rng.integers(1, 4)) for e in rng.choice(E, size=min(E, 3), replace=False)}
                          for _ in range(L)]
            plan = ReplicaPlan(capacity=C if trial % 11 else C + 1, layers=layers)
            _, placement, log = apply_batch(state, table, plan)
            batches.append({
                "assignment": a.tolist(),
                "plan_capacity": plan.capacity,
                "plan": [sorted(x.items()) for x in layers],
                "token_to_slot": [lp.token_to_slot.tolist() for lp in placement.layers],
                "slots": [[list(s) for s in lp.slots] for lp in placement.layers],
                "events": _events(log),
                "fallback_layers": list(log.fallback_layers),
            })
        out.append({"L": L, "T": T, "E": E, "capacity": C, "batches": batches})
    return out


def exec_cases():
    """Execution maps of BatchRunner._run_predicted (simulator.py:181-208), captured by
    spying _metrics_from. Predictions from an untrained SRU (so corrective loads occur)."""
    rng = np.random.default_rng(33)
    out = []
    for trial in range(150):
        L = int(rng.integers(1, 4))
        E = int(rng.integers(2, 9))
        d = int(rng.integers(4, 12))
        T = int(rng.integers(4, 40))
        shape = ModelShape(L, E, d, T)
        trace = generate_trace(shape, num_batches=4, skew=float(rng.uniform(0, 2)), seed=trial)
        C = int(rng.integers(max(1, E - 2), E + 25))
        params = init_params(L, E, d, num_sru_layers=2, seed=trial)
        runner = BatchRunner(trace, "replicated", C, params=params)
        captured = []
        orig = runner._metrics_from

        def spy(batch, execution, log, acc, _orig=orig):
            captured.append(execution)
            return _orig(batch, execution, log, acc)

        runner._metrics_from = spy
        batches = []
        for batch in trace.batches:
            outcome = runner.run_batch(batch)
            ex = captured[-1]
            batches.append({
                "predicted": outcome.table.assignment.tolist(),
                "oracle": batch.oracle_routing.tolist(),
                "exec_token_to_slot": [lp.token_to_slot.tolist() for lp in ex.layers],
                "exec_slots": [[list(s) for s in lp.slots] for lp in ex.layers],
                "placement_token_to_slot": [lp.token_to_slot.tolist() for lp in outcome.placement.layers],
                "events": _events(outcome.log),
                "fallback_layers": list(outcome.log.fallback_layers),
            })
        out.append({"L": L, "E": E, "T": T, "capacity": C, "batches": batches})
    return out


def metrics_cases():
    """simulate_strategy (src/simulator.py:268-273) per strategy, predictor and cost model:
    per-batch Metrics of the reference, with the hash tables it predicted (the GPU predictor
    is bf16, so the parity test feeds these tables and checks the cost model on its own)."""
    from dataclasses import asdict

    rng = np.random.default_rng(55)
    costs = [(1.0, 10.0, 2.0, 5.0), (1.0, 1.0, 0.1, 0.1), (0.5, 3.0, 0.0, 7.25)]
    out = []
    for trial in range(60):
        L = int(rng.integers(1, 4))
        E = int(rng.integers(2, 10))
        d = int(rng.integers(4, 12))
        T = int(rng.integers(4, 48))
        shape = ModelShape(L, E, d, T)
        hot = trial % 3 == 2
        if hot:
            nh = int(rng.integers(1, E + 1))
            trace = generate_hot_trace(shape, num_batches=4, num_hot=nh, seed=trial)
            gen = {"kind": "hot", "num_hot": nh}
        else:
            sk = float(rng.uniform(0, 2))
            trace = generate_trace(shape, num_batches=4, skew=sk, seed=trial)
            gen = {"kind": "zipf", "skew": sk}
        C = int(rng.integers(max(1, E - 2), E + 25))
        strategy = ("resident-all", "distinct-only", "replicated")[trial % 3 if trial % 5 else 2]
        cost = costs[trial % len(costs)]
        use_sru = trial % 2 == 1
        params = init_params(L, E, d, num_sru_layers=2, seed=trial) if use_sru else "oracle"
        runner = BatchRunner(trace, strategy, C, params=params, cost=CostModel(*cost))
        batches = []
        for batch in trace.batches:
            outcome = runner.run_batch(batch)
            batches.append({"table": outcome.table.assignment.tolist(), "metrics": asdict(outcome.metrics)})
        res = simulate_strategy(trace, strategy, C, params=params, cost=CostModel(*cost))
        assert [asdict(m) for m in res.per_batch] == [b["metrics"] for b in batches]
        out.append({"L": L, "E": E, "d": d, "T": T, "seed": trial, "gen": gen, "capacity": C, "strategy": strategy,
                    "cost": cost, "sru": use_sru, "batches": batches, "aggregate": asdict(res.aggregate)})
    return out


def sru_cases():
    arrays = {}
    meta = []
    rng = np.random.default_rng(44)
    specs = [(8, 16, 2, 2, 4), (16, 64, 3, 2, 6), (32, 100, 2, 3, 8), (64, 128, 4, 1, 8), (128, 256, 10, 1, 8)]
    for i, (d, T, S, L, E) in enumerate(specs):
        if i % 2 == 0:
            params = init_params(L, E, d, num_sru_layers=S, seed=100 + i)
        else:
            layers = [SruLayerParams(w=rng.normal(size=(d, d)) / np.sqrt(d), w_f=rng.normal(size=(d, d)) / np.sqrt(d),
                                     w_r=rng.normal(size=(d, d)) / np.sqrt(d), b_f=rng.normal(size=d),
                                     b_r=rng.normal(size=d)) for _ in range(S)]
            params = SruParams(layers=layers, heads=rng.normal(size=(L, E, d)))
        x = rng.normal(size=(T, d))
        h = sru_forward(x, params)
        table = predict_batch(x, params)
        key = f"c{i}"
        arrays[f"{key}_x"] = x
        arrays[f"{key}_h"] = h
        arrays[f"{key}_assign"] = table.assignment
        arrays[f"{key}_heads"] = params.heads
        entry = {"key": key, "d": d, "T": T, "S": S, "L": L, "E": E}
        if i % 2 == 0:  # init_params weights are regenerated by the oracle (predictor.py:130-154), pinned by hash
            entry["init_seed"] = 100 + i
            entry["weights_sha"] = sha(np.concatenate([np.concatenate([getattr(l, nm).ravel() for nm in
                                   ("w", "w_f", "w_r", "b_f", "b_r")]) for l in params.layers] + [params.heads.ravel()]))
            del arrays[f"{key}_heads"]
        else:
            for s, lay in enumerate(params.layers):
                for nm in ("w", "w_f", "w_r", "b_f", "b_r"):
                    arrays[f"{key}_l{s}_{nm}"] = getattr(lay, nm)
        meta.append(entry)
    return arrays, meta


def moe_cases():
    arrays = {}
    meta = []
    rng = np.random.default_rng(55)
    for i in range(40):  # acceptance criterion 1 distribution (test_acceptance.py:45-70)
        L, E, d, T = int(rng.integers(1, 5)), int(rng.integers(2, 9)), int(rng.integers(2, 17)), int(rng.integers(1, 33))
        F = int(rng.integers(2, 9))
        params = random_params(ModelShape(L, E, d, T), d_ff=F, seed=i)
        emb = rng.normal(size=(T, d)).astype(np.float32)
        routing = oracle_route_batch(emb, params)
        out = moe_forward(emb, params)
        key = f"r{i}"
        arrays.update({f"{key}_emb": emb, f"{key}_router": params.router_weights, f"{key}_u": params.expert_u,
                       f"{key}_v": params.expert_v, f"{key}_route": routing, f"{key}_out": out})
        meta.append({"key": key, "L": L, "E": E, "d": d, "T": T, "F": F})
    # config 1 of BASELINE.json: Switch layer, 8 experts, d_model 128, d_ff 512, 256 tokens, Zipf 1.2
    shape = ModelShape(1, 8, 128, 256)
    trace = generate_trace(shape, num_batches=2, skew=1.2, seed=7)
    params = oracle_params_for_trace(trace, d_ff=512)
    cfg = []
    for b, batch in enumerate(trace.batches):
        out = moe_forward(batch.embeddings, params)
        arrays[f"cfg1_b{b}_out"] = out
        arrays[f"cfg1_b{b}_route"] = batch.oracle_routing
        cfg.append({"emb_sha": sha(batch.embeddings), "route_sha": sha(batch.oracle_routing)})
    sru = init_params(1, 8, 128, num_sru_layers=10, seed=7)
    table = predict_batch(trace.batches[0], sru)
    arrays["cfg1_pred_assign"] = table.assignment
    arrays["cfg1_pred_hidden"] = sru_forward(trace.batches[0].embeddings, sru)
    params_sha = {"router": sha(params.router_weights), "u": sha(params.expert_u), "v": sha(params.expert_v)}
    return arrays, meta, {"batches": cfg, "params_sha": params_sha, "seed": 7, "skew": 1.2, "d_ff": 512,
                          "sru_seed": 7, "sru_heads_sha": sha(sru.heads)}


def workload_pins():
    pins = []
    for (L, E, d, T, nb, skew, seed) in [(2, 4, 8, 16, 5, 1.0, 7), (3, 16, 32, 200, 2, 1.2, 3), (12, 128, 64, 300, 1, 1.2, 1)]:
        tr = generate_trace(ModelShape(L, E, d, T), nb, skew, seed)
        pr = oracle_params_for_trace(tr, d_ff=2 * d)
        pins.append({"args": [L, E, d, T, nb, skew, seed], "emb": [sha(b.embeddings) for b in tr.batches],
                     "route": [sha(b.oracle_routing) for b in tr.batches],
                     "router": sha(pr.router_weights), "u": sha(pr.expert_u), "v": sha(pr.expert_v)})
    tr = generate_hot_trace(ModelShape(1, 64, 16, 64), 1, 2, 5)
    pins.append({"hot": [1, 64, 16, 64, 1, 2, 5], "route": [sha(tr.batches[0].oracle_routing)]})
    return pins


def io_files():
    """Files written by the reference's own writers (moesim-trace v1, moesim-sru-params v1,
    moesim-moe-params v1: src/workload.py:336-344, src/predictor.py:400-420,
    src/router_oracle.py:184-206) plus the arrays they hold."""
    from moesim.predictor import save_sru_params
    from moesim.router_oracle import save_params
    from moesim.workload import write_trace

    io = OUT / "io"
    io.mkdir(exist_ok=True)
    tr = generate_trace(ModelShape(2, 4, 8, 5), 2, skew=1.2, seed=3)
    write_trace(tr, io / "trace.txt")
    sp = init_params(2, 4, 8, num_sru_layers=2, seed=4)
    save_sru_params(sp, io / "sru_params.txt")
    mp = random_params(ModelShape(2, 4, 8, 5), d_ff=16, seed=5)
    save_params(mp, io / "moe_params.txt")
    arrays = {"emb": np.stack([b.embeddings for b in tr.batches]),
              "routing": np.stack([b.oracle_routing for b in tr.batches]),
              "heads": sp.heads, "router": mp.router_weights, "u": mp.expert_u, "v": mp.expert_v}
    for i, lay in enumerate(sp.layers):
        for k in ("w", "w_f", "w_r", "b_f", "b_r"):
            arrays[f"sru{i}_{k}"] = getattr(lay, k)
    np.savez_compressed(io / "io.npz", **arrays)


def training_cases():
    """Gradients and a short training run from the reference itself (src/predictor.py:238-379)."""
    from moesim.predictor import loss_and_grads, train_predictor
    from moesim.workload import RoutingTrace

    rng = np.random.default_rng(21)
    arrays = {}
    for k, (S, T, d, L, E, nl) in enumerate([(2, 5, 6, 2, 3, 2), (3, 17, 16, 1, 4, 3), (1, 64, 32, 2, 8, 2)]):
        p = init_params(L, E, d, num_sru_layers=nl, seed=k)
        x = rng.normal(size=(S, T, d))
        y = rng.integers(0, E, size=(S, L, T))
        loss, g = loss_and_grads(p, x, y)
        arrays[f"g{k}_x"], arrays[f"g{k}_y"], arrays[f"g{k}_loss"] = x, y, np.array(loss)
        arrays[f"g{k}_meta"] = np.array([S, T, d, L, E, nl, k])
        arrays[f"g{k}_heads"] = g.heads
        for i, lay in enumerate(g.layers):
            for name in ("w", "w_f", "w_r", "b_f", "b_r"):
                arrays[f"g{k}_{i}_{name}"] = getattr(lay, name)
    shape = ModelShape(num_layers=2, experts_per_layer=4, d_model=16, batch_size=32)
    tr = generate_trace(shape, num_batches=12, skew=1.2, seed=9)
    res = train_predictor(RoutingTrace(shape, tr.batches), epochs=4, learning_rate=0.01, seed=3, num_sru_layers=2,
                          sequences_per_step=5)
    arrays["t_emb"] = np.stack([b.embeddings for b in tr.batches])
    arrays["t_lab"] = np.stack([b.oracle_routing for b in tr.batches])
    arrays["t_curve"] = np.array(res.loss_curve)
    arrays["t_heads"] = res.params.heads
    for i, lay in enumerate(res.params.layers):
        for name in ("w", "w_f", "w_r", "b_f", "b_r"):
            arrays[f"t_{i}_{name}"] = getattr(lay, name)
    np.savez_compressed(OUT / "train.npz", **arrays)


def main():
    if "--only-io" in sys.argv:
        io_files()
        return
    if "--only-train" in sys.argv:
        training_cases()
        return
    if "--only-metrics" in sys.argv:
        (OUT / "metrics.json").write_text(json.dumps(metrics_cases()))
        return
    io_files()
    training_cases()
    (OUT / "planner.json").write_text(json.dumps(planner_cases()))
    (OUT / "placement.json").write_text(json.dumps(placement_cases()))
    (OUT / "exec.json").write_text(json.dumps(exec_cases()))
    (OUT / "metrics.json").write_text(json.dumps(metrics_cases()))
    arrays, meta = sru_cases()
    np.savez_compressed(OUT / "sru.npz", **arrays)
    marrays, mmeta, cfg1 = moe_cases()
    np.savez_compressed(OUT / "moe.npz", **marrays)
    (OUT / "meta.json").write_text(json.dumps({"sru": meta, "moe": mmeta, "cfg1": cfg1,
                                               "workload": workload_pins(),
                                               "reference": "arxiv/paper_2605_11537 pkg/src/moesim",
                                               "numpy": np.__version__}, indent=1))
    for p in sorted(OUT.iterdir()):
        print(p.name, p.stat().st_size)


if __name__ == "__main__":
    main()
