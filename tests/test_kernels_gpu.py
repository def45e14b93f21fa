"""Kernel-level checks of libmoempmc.so against plain PyTorch references.

These call the C-ABI directly (ctypes) on device tensors; the API-level parity
against the CPU oracle lives in test_parity_gpu.py.
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402


@pytest.fixture(scope="module")
def dev():
    return require_device()


def _rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).abs().max() / max(b.abs().max().item(), 1e-30))


@pytest.mark.parametrize(
    "M,N,K",
    [(128, 256, 64), (200, 256, 128), (1000, 384, 768), (77, 64, 64), (300, 128, 192), (4096, 2304, 768)],
)
@pytest.mark.parametrize("c_dtype", [0, 1])
def test_dense_gemm(dev, M, N, K, c_dtype):
    g = torch.Generator(device=dev).manual_seed(M * 7 + N + K)
    A = torch.randn(M, K, device=dev, generator=g).bfloat16()
    B = torch.randn(N, K, device=dev, generator=g).bfloat16()
    C = torch.zeros(M, N, device=dev, dtype=torch.bfloat16 if c_dtype == 0 else torch.float32)
    _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, c_dtype, N, None, 0, 0, stream_ptr())
    ref = A.float() @ B.float().T
    torch.cuda.synchronize()
    assert _rel(C.float(), ref) < (1e-2 if c_dtype == 0 else 1e-5)


def test_dense_gemm_bias_sigmoid_relu(dev):
    M, N, K = 257, 384, 128
    A = torch.randn(M, K, device=dev).bfloat16()
    B = torch.randn(N, K, device=dev).bfloat16()
    bias = torch.randn(N, device=dev)
    C = torch.empty(M, N, device=dev)
    _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 1, N, ptr(bias), 2, 128, stream_ptr())
    ref = A.float() @ B.float().T + bias
    ref[:, 128:] = torch.sigmoid(ref[:, 128:])
    assert _rel(C, ref) < 1e-5
    _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 1, N, None, 1, 0, stream_ptr())
    assert _rel(C, (A.float() @ B.float().T).relu()) < 1e-5


def test_histogram_and_caps(dev):
    rng = np.random.default_rng(0)
    L, T, E = 3, 1000, 37
    a = rng.integers(0, E, size=(L, T)).astype(np.int32)
    at = torch.from_numpy(a).to(dev)
    dem = torch.empty(L, E, dtype=torch.int32, device=dev)
    _lib.call("mp_histogram", ptr(at), L, T, E, ptr(dem), stream_ptr())
    ref = np.stack([np.bincount(r, minlength=E) for r in a])
    assert (dem.cpu().numpy() == ref).all()


def test_heads_argmax(dev):
    T, d, L, E, Eg = 500, 128, 3, 20, 32
    h = torch.randn(T, d, device=dev).bfloat16()
    heads = torch.zeros(((L * Eg + 63) // 64) * 64, d, device=dev)
    w = torch.randn(L, E, d, device=dev)
    for l in range(L):
        heads[l * Eg : l * Eg + E] = w[l]
    heads = heads.bfloat16()
    out = torch.full((L, T), -1, dtype=torch.int32, device=dev)
    _lib.call("mp_heads_argmax", ptr(h), ptr(heads), T, d, L, E, Eg, ptr(out), stream_ptr())
    logits = torch.einsum("td,led->lte", h.float(), heads[: L * Eg].float().view(L, Eg, d)[:, :E])
    ref = logits.argmax(-1)
    agree = (out.long() == ref).float().mean().item()
    assert agree > 0.999


def test_router_exact(dev):
    T, d, E, Eg = 1000, 128, 12, 64
    x = torch.randn(T, d, device=dev)
    w = torch.randn(E, d, device=dev)
    w[5] = w[3]  # exact tie -> lower index
    w_hi = w.bfloat16()
    w_lo = (w - w_hi.float()).bfloat16()
    whl = torch.zeros(Eg, 2 * d, device=dev, dtype=torch.bfloat16)
    whl[:E, :d] = w_hi
    whl[:E, d:] = w_lo
    route = torch.full((T,), -1, dtype=torch.int32, device=dev)
    nbytes = _lib.size_query("mp_router_workspace_bytes", T, d)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.call("mp_route_top1", ptr(x), d, T, d, ptr(whl), ptr(w), E, Eg, 0.0, ptr(route), ptr(ws), nbytes,
              stream_ptr())
    ref = (x.double() @ w.double().T).argmax(-1)
    assert (route.long() == ref).all()


@pytest.mark.parametrize("T,E", [(4096, 12), (1000, 100), (300, 64), (20000, 128)])
def test_router_histogram_path_matches(dev, T, E):
    """mp_route_top1_hist (near ties re-decided inside the router, chunk histograms written)
    + mp_exec_map_hist == mp_route_top1_ex + mp_exec_map: exact routes (forced ties) and the
    same execution map."""
    d = 128
    Eg = 64 if E <= 64 else 128
    g = torch.Generator(device=dev).manual_seed(T + 3 * E)
    x = torch.randn(T, d, device=dev, generator=g)
    w = torch.randn(E, d, device=dev, generator=g)
    w[5] = w[3]
    w[E - 1] = w[0] * (1 + 2 ** -20)
    w_hi = w.bfloat16()
    w_lo = (w - w_hi.float()).bfloat16()
    whl = torch.zeros(Eg, 2 * d, device=dev, dtype=torch.bfloat16)
    whl[:E, :d] = w_hi
    whl[:E, d:] = w_lo
    wabs = torch.empty(d, device=dev)
    _lib.call("mp_router_weight_absmax", ptr(w), E, d, ptr(wabs), stream_ptr())
    nbytes = _lib.size_query("mp_router_workspace_bytes", T, d)
    rws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ref = (x.double() @ w.double().T).argmax(-1)
    i32 = dict(dtype=torch.int32, device=dev)
    max_slots = 2 * E
    pstride = max_slots + (T + 127) // 128
    xn = _lib.size_query("mp_exec_workspace_bytes", 1, T, E, max_slots)
    outs = []
    for hist in (False, True):
        route = torch.full((T,), -7, **i32)
        o = dict(res=torch.zeros(E, **i32), tts=torch.empty(T, **i32), corr=torch.empty(E, **i32),
                 ns=torch.empty(1, **i32), rot=torch.empty(T, **i32), tor=torch.empty(T, **i32),
                 prow=torch.zeros(pstride, **i32), prows=torch.zeros(pstride, **i32), eb=torch.empty(E + 1, **i32))
        xws = torch.empty(xn, dtype=torch.uint8, device=dev)
        tail = (ptr(o["tts"]), ptr(o["corr"]), ptr(o["ns"]), ptr(o["rot"]), ptr(o["tor"]), ptr(o["prow"]),
                ptr(o["prows"]), ptr(o["eb"]))
        if hist:
            _lib.call("mp_route_top1_hist", ptr(x), d, T, d, ptr(whl), ptr(w), ptr(wabs), E, Eg, ptr(route), ptr(xws),
                      ptr(rws), nbytes, stream_ptr())
            _lib.call("mp_exec_map_hist", ptr(route), T, E, max_slots, 1, ptr(o["res"]), *tail, ptr(x), d, None,
                      ptr(xws), xn, stream_ptr())
        else:
            _lib.call("mp_route_top1_ex", ptr(x), d, T, d, ptr(whl), ptr(w), ptr(wabs), E, Eg, ptr(route), ptr(rws),
                      nbytes, stream_ptr())
            _lib.call("mp_exec_map", ptr(route), 1, T, E, max_slots, 1, ptr(o["res"]), *tail, ptr(xws), xn,
                      stream_ptr())
        torch.cuda.synchronize()
        o["route"] = route
        outs.append(o)
    a, b = outs
    assert (b["route"].long() == ref).all()
    n_pieces = int(a["eb"][-1].item())
    for k in ("route", "res", "tts", "corr", "ns", "rot", "tor", "eb"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(a["prow"][:n_pieces], b["prow"][:n_pieces])
    assert torch.equal(a["prows"][:n_pieces], b["prows"][:n_pieces])


@pytest.mark.parametrize("T,E,split_m", [(16384, 128, 1), (5000, 256, 3), (129, 7, 1), (20000, 300, 0)])
def test_exec_map_hist_from_given_chunk_histograms(dev, T, E, split_m):
    """mp_exec_map_hist (one-block chunk prefixes + layout) on chunk histograms placed in its
    workspace == mp_exec_map on the routes: E above one 128-expert column group, a warm
    residency with zeros (corrective loads), CTA-pair piece padding."""
    rng = np.random.default_rng(T + E)
    p = 1.0 / (np.arange(E) + 1.0) ** 1.1
    route_h = rng.choice(E, size=T, p=p / p.sum()).astype(np.int32)
    res0 = rng.integers(0, 3, size=E).astype(np.int32)
    route = torch.from_numpy(route_h).to(dev)
    i32 = dict(dtype=torch.int32, device=dev)
    max_slots = int(res0.sum()) + E + 1
    pstride = max_slots + (T + 127) // 128 + E
    xn = _lib.size_query("mp_exec_workspace_bytes", 1, T, E, max_slots)
    nch = (T + 127) // 128
    cc = np.zeros((nch, E), dtype=np.int32)
    np.add.at(cc, (np.arange(T) // 128, route_h), 1)
    outs = []
    for hist in (False, True):
        o = dict(res=torch.from_numpy(res0.copy()).to(dev), tts=torch.empty(T, **i32), corr=torch.empty(E, **i32),
                 ns=torch.empty(1, **i32), rot=torch.empty(T, **i32), tor=torch.empty(T, **i32),
                 prow=torch.zeros(pstride, **i32), prows=torch.zeros(pstride, **i32), eb=torch.empty(E + 1, **i32))
        xws = torch.zeros(xn, dtype=torch.uint8, device=dev)
        tail = (ptr(o["tts"]), ptr(o["corr"]), ptr(o["ns"]), ptr(o["rot"]), ptr(o["tor"]), ptr(o["prow"]),
                ptr(o["prows"]), ptr(o["eb"]))
        if hist:
            xws[: cc.nbytes].copy_(torch.from_numpy(cc.view(np.uint8).reshape(-1)))
            _lib.call("mp_exec_map_hist", ptr(route), T, E, max_slots, split_m, ptr(o["res"]), *tail, None, 1, None,
                      ptr(xws), xn, stream_ptr())
        else:
            _lib.call("mp_exec_map", ptr(route), 1, T, E, max_slots, split_m, ptr(o["res"]), *tail, ptr(xws), xn,
                      stream_ptr())
        torch.cuda.synchronize()
        outs.append(o)
    a, b = outs
    n_pieces = int(a["eb"][-1].item())
    for k in ("res", "tts", "corr", "ns", "rot", "tor", "eb"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(a["prow"][:n_pieces], b["prow"][:n_pieces])
    assert torch.equal(a["prows"][:n_pieces], b["prows"][:n_pieces])


@pytest.mark.parametrize("T,E,d", [(16384, 128, 768), (3001, 40, 1024), (200, 8, 768)])
def test_exec_map_rank_permute_matches_ffn_gather(dev, T, E, d):
    """mp_exec_map_hist with xperm (ranks + FFN permute in one kernel) == mp_exec_map_hist
    without it followed by mp_ffn_gather: same maps, same permuted bf16 rows."""
    rng = np.random.default_rng(T + E)
    p = 1.0 / (np.arange(E) + 1.0) ** 1.2
    route_h = rng.choice(E, size=T, p=p / p.sum()).astype(np.int32)
    route = torch.from_numpy(route_h).to(dev)
    x = torch.randn(T, d, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    max_slots, F = 2 * E, 256
    pstride = max_slots + (T + 127) // 128
    xn = _lib.size_query("mp_exec_workspace_bytes", 1, T, E, max_slots)
    fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
    nch = (T + 127) // 128
    cc = np.zeros((nch, E), dtype=np.int32)
    np.add.at(cc, (np.arange(T) // 128, route_h), 1)
    outs = []
    for fused in (False, True):
        o = dict(res=torch.zeros(E, **i32), tts=torch.empty(T, **i32), corr=torch.empty(E, **i32),
                 ns=torch.empty(1, **i32), rot=torch.empty(T, **i32), tor=torch.empty(T, **i32),
                 prow=torch.zeros(pstride, **i32), prows=torch.zeros(pstride, **i32), eb=torch.empty(E + 1, **i32),
                 fws=torch.zeros(fb, dtype=torch.uint8, device=dev))
        xws = torch.zeros(xn, dtype=torch.uint8, device=dev)
        xws[: cc.nbytes].copy_(torch.from_numpy(cc.view(np.uint8).reshape(-1)))
        tail = (ptr(o["tts"]), ptr(o["corr"]), ptr(o["ns"]), ptr(o["rot"]), ptr(o["tor"]), ptr(o["prow"]),
                ptr(o["prows"]), ptr(o["eb"]))
        _lib.call("mp_exec_map_hist", ptr(route), T, E, max_slots, 0, ptr(o["res"]), *tail, ptr(x), d,
                  ptr(o["fws"]) if fused else None, ptr(xws), xn, stream_ptr())
        if not fused:
            _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(o["tor"]), ptr(o["fws"]), fb, stream_ptr())
        torch.cuda.synchronize()
        outs.append(o)
    a, b = outs
    for k in ("res", "tts", "corr", "ns", "rot", "tor", "eb"):
        assert torch.equal(a[k], b[k]), k
    assert torch.equal(a["fws"][: T * d * 2], b["fws"][: T * d * 2])


def test_sru_layer_matches_fp64(dev):
    T, d = 700, 128
    g = torch.Generator().manual_seed(5)
    bound = 1.0 / np.sqrt(d)
    W = (torch.rand(3 * d, d, generator=g, dtype=torch.float64) * 2 - 1) * bound
    b = torch.zeros(3 * d, dtype=torch.float64)
    b[d:] = (torch.rand(2 * d, generator=g, dtype=torch.float64) * 2 - 1) * bound
    x = torch.randn(T, d, generator=g, dtype=torch.float64)
    # fp64 reference (src/predictor.py:157-195)
    proj = x @ W.T + b
    u, f, r = proj[:, :d], torch.sigmoid(proj[:, d:2 * d]), torch.sigmoid(proj[:, 2 * d:])
    c = torch.zeros(d, dtype=torch.float64)
    href = torch.empty_like(x)
    for t in range(T):
        c = f[t] * c + (1 - f[t]) * u[t]
        href[t] = r[t] * torch.tanh(c) + (1 - r[t]) * x[t]
    xd = x.float().to(dev)
    xb = xd.bfloat16()
    Wd = W.to(dev).bfloat16()
    bd = b.float().to(dev)
    h32 = torch.empty(T, d, device=dev)
    h16 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    nf = torch.zeros(1, dtype=torch.int32, device=dev)
    nbytes = _lib.size_query("mp_sru_workspace_bytes", T, d)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    _lib.call("mp_sru_layer", ptr(xb), ptr(xd), ptr(Wd), ptr(bd), T, d, None, ptr(h32), ptr(h16), None, ptr(nf),
              ptr(ws), nbytes, stream_ptr())
    assert int(nf.item()) == 0
    err = float((h32.double().cpu() - href).abs().max() / href.abs().max())
    assert err < 1e-2, err


@pytest.mark.parametrize("T,d", [(20000, 256), (8193, 192), (257, 64)])
def test_sru_scan_long_sequences(dev, T, d):
    """mp_sru_scan over many look-back windows (T / 256 blocks per 128-channel strip), with a
    carry-in and the final cell state, against a float64 scan of the same bf16 u/f/r."""
    g = torch.Generator().manual_seed(T)
    u = torch.randn(T, d, generator=g) * 0.5
    f = torch.sigmoid(torch.randn(T, d, generator=g) * 2 + 2)  # long memory: carries matter
    r = torch.sigmoid(torch.randn(T, d, generator=g))
    ufr = torch.cat([u, f, r], 1).bfloat16()
    x = torch.randn(T, d, generator=g)
    c0 = torch.randn(d, generator=g)
    uu, ff, rr = (v.double() for v in ufr.float().split(d, 1))
    c = c0.double()
    href = torch.empty(T, d, dtype=torch.float64)
    for t in range(T):
        c = ff[t] * c + (1 - ff[t]) * uu[t]
        href[t] = rr[t] * torch.tanh(c) + (1 - rr[t]) * x[t].double()
    nbytes = _lib.size_query("mp_sru_workspace_bytes", T, d)
    ws = torch.zeros(nbytes, dtype=torch.uint8, device=dev)
    ws[: ufr.numel() * 2].view(torch.bfloat16).copy_(ufr.reshape(-1).to(dev))
    xd, c0d = x.to(dev), c0.to(dev)
    h32 = torch.empty(T, d, device=dev)
    h16 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)
    cl = torch.empty(d, device=dev)
    nf = torch.zeros(1, dtype=torch.int32, device=dev)
    for _ in range(2):  # the second call reuses the workspace flags (reset per call)
        _lib.call("mp_sru_scan", ptr(xd), T, d, ptr(c0d), ptr(h32), ptr(h16), ptr(cl), ptr(nf), ptr(ws), nbytes,
                  stream_ptr())
        torch.cuda.synchronize()
        assert int(nf.item()) == 0
        err = float((h32.double().cpu() - href).abs().max() / href.abs().max())
        assert err < 1e-4, err
        assert float((cl.double().cpu() - c).abs().max()) < 1e-4


def test_exec_map_and_ffn(dev):
    rng = np.random.default_rng(3)
    T, E, d, F = 1500, 10, 128, 256
    route = rng.choice(E, size=T, p=np.array([0.5] + [0.5 / (E - 1)] * (E - 1))).astype(np.int32)
    res = np.zeros(E, dtype=np.int32)
    res[0] = 4  # expert 0 has 4 replicas
    res[3] = 2
    max_slots = int(res.sum()) + E
    rt = torch.from_numpy(route).to(dev)
    rs = torch.from_numpy(res).to(dev)
    i32 = dict(dtype=torch.int32, device=dev)
    tts = torch.empty(T, **i32)
    corr = torch.empty(E, **i32)
    ns = torch.empty(1, **i32)
    rot = torch.empty(T, **i32)
    tor = torch.full((T,), -1, **i32)
    pstride = max_slots + (T + 127) // 128
    prow = torch.empty(pstride, **i32)
    prows = torch.empty(pstride, **i32)
    eb = torch.empty(E + 1, **i32)
    nbytes = _lib.size_query("mp_exec_workspace_bytes", 1, T, E, max_slots)
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    for split in (0, 1):
        rs = torch.from_numpy(res).to(dev)
        _lib.call("mp_exec_map", ptr(rt), 1, T, E, max_slots, split, ptr(rs), ptr(tts), ptr(corr), ptr(ns), ptr(rot),
                  ptr(tor), ptr(prow), ptr(prows), ptr(eb), ptr(ws), nbytes, stream_ptr())
        torch.cuda.synchronize()
        # closed form F6 on host
        cnt = np.where(res > 0, res, (np.bincount(route, minlength=E) > 0).astype(np.int32))
        off = np.concatenate([[0], np.cumsum(cnt)])
        seen = np.zeros(E, dtype=np.int64)
        exp_slot = np.empty(T, dtype=np.int64)
        for t, e in enumerate(route):
            exp_slot[t] = off[e] + seen[e] % cnt[e]
            seen[e] += 1
        assert (tts.cpu().numpy() == exp_slot).all()
        assert sorted(tor.cpu().numpy().tolist()) == list(range(T))
        assert (rs.cpu().numpy() == cnt).all()
        # FFN (seeded: the tolerance below is a max over T x d elements of bf16-rounded hidden values)
        dp, Fp = d, F
        g = torch.Generator(device=dev).manual_seed(17 + split)
        U = torch.randn(E, Fp, dp, device=dev, generator=g) / np.sqrt(dp)
        V = torch.randn(E, dp, Fp, device=dev, generator=g) / np.sqrt(Fp)
        x = torch.randn(T, dp, device=dev, generator=g)
        x0 = x.clone()
        Ub, Vb = U.bfloat16().contiguous(), V.bfloat16().contiguous()
        fb = _lib.size_query("mp_ffn_workspace_bytes", T, dp, Fp)
        fws = torch.empty(fb, dtype=torch.uint8, device=dev)
        _lib.call("mp_moe_ffn", ptr(x), ptr(x), T, dp, Fp, E, ptr(Ub), ptr(Vb), ptr(tor), ptr(prow), ptr(prows), ptr(eb),
                  ptr(fws), fb, stream_ptr())
        xb = x0.bfloat16().float()
        ref = x0.clone()
        rl = torch.from_numpy(route).long().to(dev)
        for e in range(E):
            m = rl == e
            hid = (xb[m] @ Ub[e].float().T).relu().bfloat16().float()
            ref[m] += hid @ Vb[e].float().T
        # bf16 hidden values rounded on either side of a tie flip by 2^-8: 40 seeds give a
        # max of 8.4e-4 (tools/ffn_tol_probe.py); the parity bar is 1e-2
        assert _rel(x - x0, ref - x0) < 2e-3


def test_tiled_weight_layout_is_bitwise_identical(dev):
    """Pre-tiled B operands (mp_tile_kmajor) give the same bits as the reference layout."""
    rng = np.random.default_rng(11)
    T, E, d, F = 900, 6, 256, 512
    route = torch.from_numpy(rng.integers(0, E, size=T).astype(np.int32)).to(dev)
    slot_expert = torch.arange(E, dtype=torch.int32, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    tor = torch.empty(T, **i32)
    pn = E + (T + 127) // 128
    prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
    nb = _lib.size_query("mp_segments_workspace_bytes", T, E)
    sws = torch.empty(nb, dtype=torch.uint8, device=dev)
    _lib.call("mp_segments_from_slots", ptr(route), ptr(slot_expert), T, E, E, 1, ptr(tor), ptr(prow), ptr(prows),
              ptr(eb), ptr(sws), nb, stream_ptr())
    U = (torch.randn(E * F, d, device=dev) / 16).bfloat16()
    V = (torch.randn(E * d, F, device=dev) / 16).bfloat16()
    Ut, Vt = torch.empty_like(U), torch.empty_like(V)
    _lib.call("mp_tile_kmajor", ptr(U), ptr(Ut), E, F, d, _lib.size_query("mp_ffn_up_bn", F), stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(V), ptr(Vt), E, d, F, _lib.size_query("mp_ffn_down_bn", d), stream_ptr())
    x = torch.randn(T, d, device=dev)
    fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
    ws = torch.empty(fb, dtype=torch.uint8, device=dev)
    y_ref = x.clone()
    _lib.call("mp_moe_ffn", ptr(x), ptr(y_ref), T, d, F, E, ptr(U), ptr(V), ptr(tor), ptr(prow), ptr(prows), ptr(eb),
              ptr(ws), fb, stream_ptr())
    y = x.clone()
    _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())
    _lib.call("mp_ffn_up", T, d, F, E, ptr(Ut), 1, ptr(prow), ptr(prows), ptr(eb), ptr(ws), fb, stream_ptr())
    _lib.call("mp_ffn_down", ptr(y), T, d, F, E, ptr(Vt), 1, ptr(tor), ptr(prow), ptr(prows), ptr(eb), ptr(ws), fb,
              stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(y, y_ref)


@pytest.mark.parametrize("split", [1, 0])
def test_cta_pair_ffn_matches_single_cta(dev, split):
    """cta_group::2 grouped GEMMs over paired pieces == the 1-CTA kernels, bit for bit."""
    rng = np.random.default_rng(5 + split)
    T, E, d, F = 3000, 9, 256, 512
    p = 1.0 / (np.arange(E) + 1.0) ** 1.3
    route = torch.from_numpy(rng.choice(E, size=T, p=p / p.sum()).astype(np.int32)).to(dev)
    slot_expert = torch.arange(E, dtype=torch.int32, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    nb = _lib.size_query("mp_segments_workspace_bytes", T, E)
    sws = torch.empty(nb, dtype=torch.uint8, device=dev)
    pn = 2 * (E + (T + 127) // 128)

    def segments(flags):
        tor = torch.empty(T, **i32)
        prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
        _lib.call("mp_segments_from_slots", ptr(route), ptr(slot_expert), T, E, E, flags, ptr(tor), ptr(prow),
                  ptr(prows), ptr(eb), ptr(sws), nb, stream_ptr())
        return tor, prow, prows, eb

    U = (torch.randn(E * F, d, device=dev) / 16).bfloat16()
    V = (torch.randn(E * d, F, device=dev) / 22).bfloat16()
    Ut, Vt = torch.empty_like(U), torch.empty_like(V)
    _lib.call("mp_tile_kmajor", ptr(U), ptr(Ut), E, F, d, 256, stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(V), ptr(Vt), E, d, F, 256, stream_ptr())
    x = torch.randn(T, d, device=dev)
    fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
    ws = torch.empty(fb, dtype=torch.uint8, device=dev)

    def run(flags_seg, flags_ffn, u, v):
        tor, prow, prows, eb = segments(flags_seg)
        y = x.clone()
        _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())
        _lib.call("mp_ffn_up", T, d, F, E, ptr(u), flags_ffn, ptr(prow), ptr(prows), ptr(eb), ptr(ws), fb,
                  stream_ptr())
        _lib.call("mp_ffn_down", ptr(y), T, d, F, E, ptr(v), flags_ffn, ptr(tor), ptr(prow), ptr(prows), ptr(eb),
                  ptr(ws), fb, stream_ptr())
        torch.cuda.synchronize()
        return y, eb

    y1, _ = run(split, 0, U, V)
    y2, eb = run(split | 2, 3, Ut, Vt)
    assert (eb.cpu().numpy() % 2 == 0).all()
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("skew,d,F", [(0.0, 256, 768), (1.2, 512, 512), (1.2, 768, 3072), (8.0, 768, 1280)])
def test_single_cta_gemm2_reads_pair_tiled_v(dev, skew, d, F):
    """flags bit 6: the single-CTA GEMM2 reading V tiled in 256-column slices (the CTA-pair
    layout; expert parallelism reuses the weights of a pair-mode pipeline) == the reference
    layout, bit for bit."""
    _check_ffn_mode_bitwise(dev, skew, d, F, 1, 64)


def _check_ffn_mode_bitwise(dev, skew, d, F, tiled, mode):
    """mp_ffn_gather / up / down with ``mode`` flags == mp_moe_ffn on the reference layout, bit for
    bit: odd and even piece counts per expert, empty experts."""
    rng = np.random.default_rng(int(skew * 10) + d + F)
    T, E = 5000, 21
    p = 1.0 / (np.arange(E) + 1.0) ** skew
    p[E // 2] = 0.0  # an expert with no tokens
    route = torch.from_numpy(rng.choice(E, size=T, p=p / p.sum()).astype(np.int32)).to(dev)
    slot_expert = torch.arange(E, dtype=torch.int32, device=dev)
    i32 = dict(dtype=torch.int32, device=dev)
    nb = _lib.size_query("mp_segments_workspace_bytes", T, E)
    sws = torch.empty(nb, dtype=torch.uint8, device=dev)
    pn = E + (T + 127) // 128
    tor = torch.empty(T, **i32)
    prow, prows, eb = torch.empty(pn, **i32), torch.empty(pn, **i32), torch.empty(E + 1, **i32)
    _lib.call("mp_segments_from_slots", ptr(route), ptr(slot_expert), T, E, E, 1, ptr(tor), ptr(prow), ptr(prows),
              ptr(eb), ptr(sws), nb, stream_ptr())
    U = (torch.randn(E * F, d, device=dev) / 16).bfloat16()
    V = (torch.randn(E * d, F, device=dev) / 28).bfloat16()
    if tiled:  # V column tiles: 256 with bit 6, else mp_ffn_down_bn
        vbn = 256 if mode & 64 else _lib.size_query("mp_ffn_down_bn", d)
        Ut, Vt = torch.empty_like(U), torch.empty_like(V)
        _lib.call("mp_tile_kmajor", ptr(U), ptr(Ut), E, F, d, _lib.size_query("mp_ffn_up_bn", F), stream_ptr())
        _lib.call("mp_tile_kmajor", ptr(V), ptr(Vt), E, d, F, vbn, stream_ptr())
    else:
        Ut, Vt = U, V
    x = torch.randn(T, d, device=dev)
    fb = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
    ws = torch.empty(fb, dtype=torch.uint8, device=dev)
    y1 = x.clone()
    _lib.call("mp_moe_ffn", ptr(x), ptr(y1), T, d, F, E, ptr(U), ptr(V), ptr(tor), ptr(prow), ptr(prows), ptr(eb),
              ptr(ws), fb, stream_ptr())
    h0 = (T * d * 2 + 255) // 256 * 256  # hidden buffer offset in the FFN workspace
    h1 = ws[h0:h0 + T * F * 2].clone()
    y2 = x.clone()
    ws.zero_()
    _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(tor), ptr(ws), fb, stream_ptr())
    _lib.call("mp_ffn_up", T, d, F, E, ptr(Ut), tiled | (mode & 2), ptr(prow), ptr(prows), ptr(eb), ptr(ws), fb,
              stream_ptr())
    h2 = ws[h0:h0 + T * F * 2].clone()
    _lib.call("mp_ffn_down", ptr(y2), T, d, F, E, ptr(Vt), tiled | mode, ptr(tor), ptr(prow), ptr(prows), ptr(eb),
              ptr(ws), fb, stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(h1, h2)
    assert torch.equal(y1, y2)


@pytest.mark.parametrize("E,d,T", [(16, 768, 5000), (64, 512, 5000), (128, 768, 16384), (4, 1024, 3000),
                                   (100, 768, 2000)])
def test_router_exact_on_dense_random_inputs(dev, E, d, T):
    """Routing equals the float64 argmax (first index on ties) on inputs whose every
    coordinate matters (random x and W, all k-blocks contribute): the fused router's x ring
    was once handed back to its TMA producer before its generic loads had read the slot,
    which corrupted whole k-blocks of some rows -- invisible on the synthetic workload, whose
    router rows are zero in half the dimensions. Both router entry points, several calls."""
    from paper_2605_11537_b200.router_oracle import ToyMoeParams, _device_moe

    rng = np.random.default_rng(E + d)
    W = rng.normal(size=(1, E, d)).astype(np.float32)
    lay = _device_moe(ToyMoeParams(W, np.zeros((1, E, 256, d), np.float32), np.zeros((1, E, d, 256), np.float32)),
                      dev).layers[0]
    e0 = rng.choice(E, size=T)
    x = torch.from_numpy((W[0][e0] * 0.05 + rng.normal(size=(T, d)) * 0.5).astype(np.float32)).to(dev)
    ref = (x.double() @ torch.from_numpy(W[0]).to(dev).double().T).argmax(1).int()
    rb = _lib.size_query("mp_router_workspace_bytes", T, d)
    ws = torch.empty(rb, dtype=torch.uint8, device=dev)
    route = torch.empty(T, dtype=torch.int32, device=dev)
    hist = torch.empty((T + 127) // 128 * E, dtype=torch.int32, device=dev)
    for _ in range(3):
        _lib.call("mp_route_top1_ex", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                  ptr(route), ptr(ws), rb, stream_ptr())
        torch.cuda.synchronize()
        assert torch.equal(route, ref)
        if lay.Eg <= 128:
            _lib.call("mp_route_top1_hist", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                      ptr(route), ptr(hist), ptr(ws), rb, stream_ptr())
            torch.cuda.synchronize()
            assert torch.equal(route, ref)
            counts = torch.bincount(ref[:(T // 128) * 128].long(), minlength=E)
            assert torch.equal(hist[:(T // 128) * E].view(-1, E).sum(0).long(), counts)
