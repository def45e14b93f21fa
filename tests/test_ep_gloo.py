"""Expert parallelism across processes on the CPU (gloo): the EP orchestrator
(paper_2605_11537_b200/ep.py -- all-gather of counts, plan, variable
all-to-all dispatch and combine) with the numpy oracle kernels must reproduce
the single-device execution map (src/simulator.py:185-203) and MoE forward
(src/router_oracle.py:119-135) exactly."""

import socket
import sys
from pathlib import Path

import numpy as np
import pytest
import torch.multiprocessing as mp

sys.path.insert(0, str(Path(__file__).resolve().parent))

from oracle import moesim_oracle as O  # noqa: E402
from oracle.ep_oracle import bf16_round, ep_plan  # noqa: E402
import ep_worker  # noqa: E402


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def single_device(seed):
    router, eu, ev, x, res = ep_worker.make_problem(seed)
    x = x.copy()
    res = res.astype(np.int64)
    slots = []
    for l in range(router.shape[0]):
        route = np.array([O.route_top1(router[l], x[t]) for t in range(x.shape[0])])
        tts, res[l], _ = O.exec_map(res[l], route)
        slots.append(tts)
        xb = bf16_round(x)
        for t in range(x.shape[0]):
            x[t] = x[t] + O.expert_forward(xb[t], eu[l, route[t]], ev[l, route[t]])
    return x, res, np.stack(slots)


@pytest.mark.parametrize("world", [2, 3])
def test_expert_parallel_matches_single_device(tmp_path, world):
    seed = 7
    mp.spawn(ep_worker.run_worker, args=(world, free_port(), seed, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"{r}.npz") for r in range(world)]
    x_ref, res_ref, slots_ref = single_device(seed)
    x_ep = np.concatenate([o["x"] for o in outs])
    slots_ep = np.concatenate([o["slots"] for o in outs], axis=1)
    assert (slots_ep == slots_ref).all()  # global stable ranks == single-device slots
    for o in outs:
        assert (o["res"] == res_ref).all()  # replicated residency state stays identical
    assert x_ep.tobytes() == x_ref.tobytes()  # dispatch + combine are exact


def test_plan_conservation_and_balance():
    """Row counts: every token sent exactly once; per-rank send/recv matrices are consistent."""
    rng = np.random.default_rng(3)
    for _ in range(50):
        G, E = int(rng.integers(1, 9)), int(rng.integers(2, 40))
        T = int(rng.integers(1, 300))
        routes = [rng.integers(0, E, size=T) for _ in range(G)]
        C = np.stack([np.bincount(r, minlength=E) for r in routes])
        res0 = rng.integers(0, 5, size=E)
        plans = [ep_plan(routes[r], C, res0.copy(), r) for r in range(G)]
        send = np.stack([p["send_counts"] for p in plans])  # send[r][d]
        recv = np.stack([p["recv_counts"] for p in plans])  # recv[d][r]
        assert (send == recv.T).all()
        for r in range(G):
            assert sorted(plans[r]["send_pos"].tolist()) == list(range(T))
            assert plans[r]["n_local"] == recv[r].sum()
