"""numpy restatement of the expert-parallel kernels (paper_2605_11537_b200/csrc/ep.cu)
-- TEST INFRASTRUCTURE for the CPU multi-process (gloo) tests of ``ep.py``.

Same contracts as ``CudaEpKernels``; the expert FFN is the reference's
per-token float32 ``v @ relu(u @ x)`` (src/router_oracle.py:101-111) applied to
bf16-rounded rows, and routing is the reference's float64 argmax
(src/router_oracle.py:90-98). Dispatch buffers are float32 holding the
bf16-rounded values (gloo-friendly).
"""

from __future__ import annotations

import numpy as np
import torch

from . import moesim_oracle as O


def _F(x, j, c):
    return np.where(x > j, (x - j + c - 1) // c, 0)


def ep_plan(route, C, res, rank, split=True):
    """Plan for one rank: mirrors k_ep_plan / k_ep_send_pos. C: (G, E) int; res: (E,) int (updated)."""
    route = np.asarray(route, dtype=np.int64)
    C = np.asarray(C, dtype=np.int64)
    G, E = C.shape
    n = C.sum(0)
    B = C[:rank].sum(0)
    cnt = np.where(res > 0, res, (n > 0).astype(np.int64))
    res[:] = cnt
    off = np.concatenate([[0], np.cumsum(cnt)])
    S = int(off[-1])
    slot_e = np.repeat(np.arange(E), cnt)
    slot_j = np.arange(S) - off[slot_e]
    slot_c = cnt[slot_e]
    acc = np.concatenate([np.zeros((1, E), np.int64), np.cumsum(C, 0)])  # (G+1, E)
    rows = np.stack([_F(acc[g + 1][slot_e], slot_j, slot_c) - _F(acc[g][slot_e], slot_j, slot_c) for g in range(G)])
    size = rows.sum(0)
    # slot list cut into G blocks of equal rows (the slot's row midpoint decides its GPU)
    before = np.concatenate([[0], np.cumsum(size)[:-1]]) if S else np.zeros(0, np.int64)
    total = int(size.sum())
    slot_gpu = np.minimum(G - 1, ((2 * before + size) * G) // (2 * total)) if total > 0 else np.zeros(S, np.int64)
    # sender
    send_counts = np.array([rows[rank][slot_gpu == dd].sum() for dd in range(G)], dtype=np.int64)
    send_displ = np.concatenate([[0], np.cumsum(send_counts)])
    send_base = np.zeros(S, np.int64)
    for dd in range(G):
        idx = np.nonzero(slot_gpu == dd)[0]
        send_base[idx] = send_displ[dd] + np.concatenate([[0], np.cumsum(rows[rank][idx])])[:-1]
    lr = O.stable_rank(route, E) if route.size else np.zeros(0, np.int64)
    grank = B[route] + lr
    c = cnt[route]
    j = grank % np.maximum(c, 1)
    s = off[route] + j
    send_pos = send_base[s] + grank // c - _F(B[route], j, c)
    # receiver
    hosted = np.nonzero(slot_gpu == rank)[0]
    recv_counts = np.array([rows[g][hosted].sum() for g in range(G)], dtype=np.int64)
    recv_displ = np.concatenate([[0], np.cumsum(recv_counts)])
    local_base = np.concatenate([[0], np.cumsum(size[hosted])])
    n_local = int(local_base[-1])
    recv_of_local = np.zeros(n_local, np.int64)
    for hi, sl in enumerate(hosted):
        lstart = local_base[hi]
        for g in range(G):
            r0 = recv_displ[g] + rows[g][hosted[:hi]].sum()
            m = rows[g][sl]
            recv_of_local[lstart:lstart + m] = r0 + np.arange(m)
            lstart += m
    pieces = []  # (expert, local row, rows) per hosted slot, M-tiles of <= 128 rows
    for hi, sl in enumerate(hosted):
        sz = int(size[sl])
        for p in range(0, sz, 128) if split else [0]:
            if sz:
                pieces.append((int(slot_e[sl]), int(local_base[hi] + p), min(128, sz - p) if split else sz))
    return dict(send_counts=send_counts, recv_counts=recv_counts, send_pos=send_pos, recv_of_local=recv_of_local,
                n_local=n_local, slot_of_token=s, pieces=pieces, slot_gpu=slot_gpu)


def bf16_round(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).bfloat16().float().numpy()


class OracleEpKernels:
    """CPU stand-in for CudaEpKernels (tests only)."""

    dispatch_dtype = torch.float32
    dev = "cpu"

    def __init__(self, router, eu, ev, rank, world):
        self.router, self.eu, self.ev = router, eu, ev  # (L,E,d), (L,E,F,d), (L,E,d,F) float32
        self.rank, self.G = rank, world
        self.E = router.shape[1]
        self.d = router.shape[2]

    def route(self, x, l):
        xs = x.numpy()
        return torch.from_numpy(np.array([O.route_top1(self.router[l], xs[t]) for t in range(xs.shape[0])],
                                         dtype=np.int32))

    def counts(self, route):
        return torch.from_numpy(np.bincount(route.numpy(), minlength=self.E).astype(np.int32))

    def plan(self, route, C, res):
        r = res.numpy().astype(np.int64)
        p = ep_plan(route.numpy(), C.numpy(), r, self.rank)
        res.copy_(torch.from_numpy(r.astype(np.int32)))
        self._p = p
        from paper_2605_11537_b200.ep import EpPlan

        return EpPlan(p["send_counts"].tolist(), p["recv_counts"].tolist(), p["n_local"],
                      torch.from_numpy(p["send_pos"]), None, None, None)

    def pack(self, x, plan, n_send):
        buf = np.zeros((n_send, self.d), np.float32)
        buf[plan.send_pos.numpy()] = bf16_round(x.numpy())
        return torch.from_numpy(buf)

    def expert_ffn(self, recvbuf, plan, l):
        p = self._p
        rb = recvbuf.numpy()
        y = np.zeros_like(rb)
        for e, row0, nrows in p["pieces"]:
            for r in range(row0, row0 + nrows):
                ri = p["recv_of_local"][r]
                y[ri] = O.expert_forward(rb[ri], self.eu[l, e], self.ev[l, e])
        return torch.from_numpy(y)

    def combine(self, x, yback, plan):
        xs = x.numpy()
        xs += yback.numpy()[plan.send_pos.numpy()]
