"""Device-resident MoE-MPMC inference pipeline (the benchmarked hot path).

One batch ("step") = the paper's Alg. 2 + Alg. 1 + the MoE forward, all on the
GPU with no host synchronisation (reference call stack: src/simulator.py:127-208
driving src/predictor.py:212-223, src/planner.py:27-85, src/placement.py:109-180,
src/router_oracle.py:119-135):

  1. predict    S SRU layers over the batch token sequence + per-layer head argmax
                (mp_sru_layer x S, mp_heads_argmax)                -> pred (L, T)
  2. plan+place histogram -> capped replica plan -> residency update / token walk
                for all L layers (mp_histogram_ws, mp_cap_replicas, mp_place)
  3. forward    per MoE layer: true top-1 routing (mp_route_top1_ex), execution
                map onto the resident replicas + corrective loads + replica-segment
                permutation (mp_exec_map), gather, grouped expert GEMM1 (+ReLU),
                grouped GEMM2 with scatter + residual combine (mp_ffn_*).

Replication modes (SURVEY.md §7 baselines):
  "off"   distinct-only caps (one replica per demanded expert), each replica's
          rows are one serial work unit  -> the non-replicated GPU baseline (ii)
  "on"    capped replica plan (demand in M-tiles by default),
          each replica one work unit                                     (iii)
  "split" like "on" but every 128-row M-tile is its own work unit (upper bound)
"""

from __future__ import annotations

import ctypes
import dataclasses
import math
from dataclasses import asdict, dataclass

import torch

from . import _lib
from ._dev import ptr, require_device, round_up, stream_ptr
from .predictor import DeviceSru
from .router_oracle import DeviceMoeLayer, router_eg

DISTINCT_ONLY_UNIT = 1 << 30  # ceil(n / unit) == 1 for every demanded expert


@dataclass
class PipelineConfig:
    num_layers: int = 12          # Switch-base MoE layers
    num_experts: int = 128        # Switch-base-128
    d_model: int = 768
    d_ff: int = 3072
    tokens: int = 16384           # tokens per batch (per GPU)
    sru_layers: int = 10          # src/predictor.py:19
    capacity: int = 296           # replica slots per layer (2 x 148 SMs)
    demand_unit: int = 128        # 1 = reference token demand; 128 = M-tile demand (F12)
    replication: str = "on"       # on | off | split
    predictor: str = "constructed"  # constructed (highway-open SRU, heads = router rows) | random
    ffn: str = "auto"             # auto (pair at >= 1024 tokens/expert, else two) | two (single-CTA
                                  # grouped GEMMs) | pair (CTA-pair cta_group::2 grouped GEMMs)
    skew: float = 1.2
    noise: float = 0.1
    physical_replicas: bool = False  # every replica slot owns a copy of its expert's weights (K9):
                                  # LOAD / REPLICATE / OFFLOAD copy weights in a per-layer pool; off:
                                  # replicas on one GPU alias the expert's single copy
    seed: int = 0                 # model: routers, experts, predictor (identical on every rank)
    batch_seed: int | None = None  # synthetic batches (per rank under EP); None: derived from seed

    def as_dict(self):
        return asdict(self)


class SyntheticSwitch:
    """Device-side synthetic Switch-base workload with the reference's distributions
    (src/workload.py:123-313): unit expert centroids in the first d/2 "routing"
    dimensions, Zipf(skew) popularity over a seeded permutation, a seeded expert
    permutation per layer, embeddings = centroid + N(0, noise^2) resampled until
    the router margin is >= 0.02, router rows = permuted centroids, U ~ N(0, 1/d),
    V ~ N(0, 1/F) with the routing rows of V zeroed (so routing is reproducible)."""

    MARGIN = 0.02

    def __init__(self, cfg: PipelineConfig, device: torch.device):
        self.cfg = cfg
        self.dev = device
        g = torch.Generator(device=device).manual_seed(cfg.seed)
        self.g = g  # model draws (same on every rank)
        bseed = cfg.batch_seed if cfg.batch_seed is not None else cfg.seed * 1000003 + 17
        self.gb = torch.Generator(device=device).manual_seed(bseed)  # batch draws
        E, d, L = cfg.num_experts, cfg.d_model, cfg.num_layers
        self.k = max(1, d // 2)
        c = torch.randn(E, self.k, device=device, generator=g, dtype=torch.float64)
        c = c / c.norm(dim=1, keepdim=True)
        self.centroids = torch.zeros(E, d, device=device)
        self.centroids[:, : self.k] = c.float()
        rank = torch.empty(E, dtype=torch.long, device=device)
        rank[torch.randperm(E, device=device, generator=g)] = torch.arange(E, device=device)
        w = 1.0 / (rank.double() + 1.0) ** cfg.skew
        self.probs = (w / w.sum()).float()
        perms = [torch.arange(E, device=device)]
        for _ in range(1, L):
            perms.append(torch.randperm(E, device=device, generator=g))
        self.perms = torch.stack(perms)  # (L, E): expert at layer l of layer-0 expert e

    def router(self, l: int) -> torch.Tensor:
        r = torch.empty_like(self.centroids)
        r[self.perms[l]] = self.centroids
        return r

    def expert_weights(self, l: int):
        cfg = self.cfg
        E, d, F = cfg.num_experts, cfg.d_model, cfg.d_ff
        u = torch.empty(E, F, d, device=self.dev, dtype=torch.bfloat16)
        v = torch.empty(E, d, F, device=self.dev, dtype=torch.bfloat16)
        for e in range(E):  # per expert to bound the fp32 temporaries
            u[e] = (torch.randn(F, d, device=self.dev, generator=self.g) / math.sqrt(d)).to(torch.bfloat16)
            ve = torch.randn(d, F, device=self.dev, generator=self.g) / math.sqrt(F)
            ve[: self.k] = 0.0
            v[e] = ve.to(torch.bfloat16)
        return u, v

    def batch(self, T: int):
        """(embeddings (T, d) fp32, layer-0 experts (T,), oracle routing (L, T))."""
        e0 = torch.multinomial(self.probs, T, replacement=True, generator=self.gb)
        base = self.centroids[e0]
        emb = torch.empty_like(base)
        pending = torch.arange(T, device=self.dev)
        rout = self.centroids[:, : self.k].double()
        for _ in range(100):
            cand = base[pending] + self.cfg.noise * torch.randn(len(pending), self.cfg.d_model, device=self.dev,
                                                                generator=self.gb)
            logits = cand[:, : self.k].double() @ rout.T
            own = logits.gather(1, e0[pending, None]).squeeze(1)
            logits.scatter_(1, e0[pending, None], -math.inf)
            ok = own - logits.max(dim=1).values >= self.MARGIN
            emb[pending[ok]] = cand[ok]
            pending = pending[~ok]
            if len(pending) == 0:
                break
        return emb, e0, self.perms[:, e0]


class MoEPipeline:
    """Weights + buffers resident in HBM; ``step`` runs one batch with zero host syncs."""

    def __init__(self, cfg: PipelineConfig, device: torch.device | None = None, workload: SyntheticSwitch | None = None):
        if cfg.ffn == "auto":
            # CTA-pair grouped GEMMs once the layer is compute-heavy (>= 1024 tokens per expert:
            # BASELINE config 2 runs at 1,126 vs 1,007 TF/s); single-CTA units on weight-streaming
            # layers (config 3: 128 tokens per expert, pairs are 12 % slower) -- profiles/README.md
            pair = cfg.tokens >= 1024 * cfg.num_experts and cfg.d_model % 256 == 0
            cfg = dataclasses.replace(cfg, ffn="pair" if pair else "two")
        self.cfg = cfg
        self.dev = device or require_device()
        dev = self.dev
        L, E, d, F, T = cfg.num_layers, cfg.num_experts, cfg.d_model, cfg.d_ff, cfg.tokens
        assert d % 64 == 0 and F % 256 == 0, "engine expects Switch-base-like padded sizes"
        self.wl = workload or SyntheticSwitch(cfg, dev)
        self.dp, self.Fp = d, F
        # ---- MoE layers (bf16 expert weights, split-bf16 router)
        self.layers = []
        for l in range(L):
            u, v = self.wl.expert_weights(l)
            self.layers.append(DeviceMoeLayer.from_device(self.wl.router(l), u, v, cfg.ffn))
        # ---- predictor (S SRU layers + heads)
        g = torch.Generator(device=dev).manual_seed(cfg.seed + 1)
        bound = 1.0 / math.sqrt(d)

        def draw(*shape):
            return (torch.rand(*shape, device=dev, generator=g, dtype=torch.float64) * 2 - 1) * bound

        sru = []
        for _ in range(cfg.sru_layers):
            w, w_f, w_r, b_f, b_r = draw(d, d), draw(d, d), draw(d, d), draw(d), draw(d)
            if cfg.predictor == "constructed":
                b_r = b_r - 8.0  # highway-open: h ~= x, so heads = router rows forecast the routing
            sru.append((w, w_f, w_r, b_f, b_r))
        if cfg.predictor == "constructed":
            heads = torch.stack([self.wl.router(l) for l in range(L)]).double()
        else:
            heads = draw(L, E, d)
        # host float64 copies: the checks in tests/ and bench.py recompute the predictor from them
        self.sru_host = [tuple(t.cpu().numpy() for t in lay) for lay in sru]
        self.heads_host = heads.cpu().numpy()
        self.sru = DeviceSru(self.sru_host, self.heads_host, dev)
        # ---- buffers
        i32 = dict(dtype=torch.int32, device=dev)
        self.assign = torch.empty(L, T, **i32)
        self.demand = torch.empty(L, E, **i32)
        self.caps = torch.empty(L, E, **i32)
        self.infeasible = torch.empty(L, **i32)
        self.res = torch.zeros(L, E, **i32)
        self.pred_slot = torch.empty(L, T, **i32)
        self.pred_event = torch.empty(L, T, **i32)
        self.offloads = torch.empty(L, E, **i32)
        self.fallback = torch.empty(L, **i32)
        self.num_slots = torch.empty(L, **i32)
        self.route = torch.empty(L, T, **i32)
        self.max_slots = max(cfg.capacity, E) + E  # placement / execution slots of one device
        self.exec_slot = torch.empty(L, T, **i32)
        self.corrective = torch.empty(L, E, **i32)
        self.exec_slots = torch.empty(L, **i32)
        self.tok_of_row = torch.empty(L, T, **i32)
        pstride = self.max_slots + (T + 127) // 128
        self.piece_row = torch.empty(L, pstride, **i32)
        self.piece_rows = torch.empty(L, pstride, **i32)
        self.exp_begin = torch.empty(L, E + 1, **i32)
        self.nonfinite = torch.zeros(1, **i32)
        self.h32 = [torch.empty(T, d, device=dev) for _ in range(2)]
        self.h16 = [torch.empty(T, d, device=dev, dtype=torch.bfloat16) for _ in range(2)]
        self.x16 = torch.empty(T, d, device=dev, dtype=torch.bfloat16)

        def ws(n):
            return torch.empty(max(int(n), 256), dtype=torch.uint8, device=dev)

        self.ws_sru_n = _lib.size_query("mp_sru_workspace_bytes", T, d)
        self.ws_sru = ws(self.ws_sru_n)
        self.ws_hist_n = _lib.size_query("mp_histogram_workspace_bytes", L, T, E)
        self.ws_hist = ws(self.ws_hist_n)
        self.ws_place_n = _lib.size_query("mp_place_workspace_bytes", L, T, E)
        self.ws_place = ws(self.ws_place_n)
        self.ws_exec_n = _lib.size_query("mp_exec_workspace_bytes", 1, T, E, self.max_slots)
        self.ws_exec = ws(self.ws_exec_n)
        self.ws_router_n = _lib.size_query("mp_router_workspace_bytes", T, d)
        self.ws_router = ws(self.ws_router_n)
        self.ws_ffn_n = _lib.size_query("mp_ffn_workspace_bytes", T, d, F)
        self.ws_ffn = ws(self.ws_ffn_n)
        self.pstride = pstride
        self.launches_per_step = None
        if cfg.physical_replicas:
            self._init_replica_pools()

    def _init_replica_pools(self) -> None:
        """Per-layer pools of P = max_slots expert-sized weight slots (K9, csrc/replica.cu)."""
        from .errors import ConfigurationError

        cfg = self.cfg
        if cfg.ffn != "two":
            raise ConfigurationError("physical replicas run on the single-CTA grouped GEMMs (ffn='two')")
        E, d, F = cfg.num_experts, self.dp, self.Fp
        self.pool_P = self.max_slots
        self.pool_R = self.max_slots
        nb = _lib.size_query("mp_pool_state_bytes", E, self.pool_R, self.pool_P)
        self.pool_state, self.pool_u, self.pool_v = [], [], []
        sp = stream_ptr()
        for l in range(cfg.num_layers):
            st = torch.empty(nb, dtype=torch.uint8, device=self.dev)
            _lib.call("mp_pool_init", E, self.pool_R, self.pool_P, ptr(st), sp)
            self.pool_state.append(st)
            self.pool_u.append(torch.empty(self.pool_P * F, d, dtype=torch.bfloat16, device=self.dev))
            self.pool_v.append(torch.empty(self.pool_P * d, F, dtype=torch.bfloat16, device=self.dev))
        self.piece_wbase = torch.zeros(cfg.num_layers, self.pstride, dtype=torch.int32, device=self.dev)
        self.pool_stats = torch.zeros(cfg.num_layers, 4, dtype=torch.int32, device=self.dev)

    def replica_stats(self) -> dict:
        """Copies since the pools were created: {loads, replicates, offloads, bytes, overflow}."""
        if not self.cfg.physical_replicas:
            return {}
        sp = stream_ptr()
        for l in range(self.cfg.num_layers):
            _lib.call("mp_pool_stats", ptr(self.pool_state[l]), self.cfg.num_experts, self.pool_R, self.pool_P,
                      ptr(self.pool_stats[l]), sp)
        s = self.pool_stats.sum(0).tolist()
        return {"loads": s[0], "replicates": s[1], "offloads": s[2],
                "bytes": (s[0] + s[1]) * self.expert_weight_bytes(), "overflow": bool(s[3])}

    # ------------------------------------------------------------------ pieces of a step
    def predict(self, x: torch.Tensor, sp: int) -> int:
        """Alg. 2: SRU stack over the batch sequence, head argmax -> self.assign. Returns #launches."""
        cfg, T, d = self.cfg, self.cfg.tokens, self.dp
        n = 0
        _lib.call("mp_f32_to_bf16", ptr(x), ptr(self.x16), T * d, sp)
        n += 1
        cur32, cur16 = x, self.x16
        for i, (W, B) in enumerate(zip(self.sru.w_cat, self.sru.b_cat)):
            h32, h16 = self.h32[i % 2], self.h16[i % 2]
            _lib.call("mp_sru_layer", ptr(cur16), ptr(cur32), ptr(W), ptr(B), T, d, None, ptr(h32), ptr(h16), None,
                      ptr(self.nonfinite), ptr(self.ws_sru), self.ws_sru_n, sp)
            n += 2  # projection GEMM + single-pass scan
            cur32, cur16 = h32, h16
        _lib.call("mp_heads_argmax", ptr(cur16), ptr(self.sru.heads), T, d, cfg.num_layers, cfg.num_experts,
                  self.sru.Eg, ptr(self.assign), sp)
        return n + 1

    def plan_and_place(self, sp: int) -> int:
        """Alg. 1: demand histogram -> capped plan -> residency + token walk for all layers."""
        cfg, L, T, E = self.cfg, self.cfg.num_layers, self.cfg.tokens, self.cfg.num_experts
        unit = DISTINCT_ONLY_UNIT if cfg.replication == "off" else cfg.demand_unit
        _lib.call("mp_histogram_ws", ptr(self.assign), L, T, E, ptr(self.demand), ptr(self.ws_hist), self.ws_hist_n,
                  sp)
        _lib.call("mp_cap_replicas", ptr(self.demand), L, E, cfg.capacity, unit, ptr(self.caps),
                  ptr(self.infeasible), sp)
        _lib.call("mp_place", ptr(self.assign), L, T, E, ptr(self.caps), cfg.capacity, cfg.capacity, ptr(self.res),
                  ptr(self.pred_slot), ptr(self.pred_event), ptr(self.offloads), ptr(self.fallback),
                  ptr(self.num_slots), ptr(self.ws_place), self.ws_place_n, sp)
        return 2 + 1 + 4

    def layer(self, l: int, x: torch.Tensor, sp: int, ev=None) -> int:
        """One MoE layer in place on the residual stream x. Returns #kernel launches.

        ev: optional 3 events recorded around GEMM1 / GEMM2 (roofline timing)."""
        cfg, T, E, d, F = self.cfg, self.cfg.tokens, self.cfg.num_experts, self.dp, self.Fp
        lay = self.layers[l]
        use_pair = cfg.ffn == "pair" and d % 256 == 0
        # replication "off" keeps one serial unit per replica (one server per expert, the paper's
        # baseline); "split" makes every 128-row tile its own unit; the CTA-pair kernels need
        # <= 128-row pieces padded to an even count per expert (split_m = 3)
        split = 3 if use_pair else (1 if cfg.replication == "split" else 0)
        # the permute into the FFN workspace rides on the execution map's rank kernel
        gather_fused = d in (768, 1024)
        if lay.Eg <= 128:
            # the router re-decides near ties itself (float64) and writes each 128-token tile's
            # expert histogram into the execution-map workspace: routing + histogram in one launch
            _lib.call("mp_route_top1_hist", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                      ptr(self.route[l]), ptr(self.ws_exec), ptr(self.ws_router), self.ws_router_n, sp)
            _lib.call("mp_exec_map_hist", ptr(self.route[l]), T, E, self.max_slots, split, ptr(self.res[l]),
                      ptr(self.exec_slot[l]), ptr(self.corrective[l]), ptr(self.exec_slots[l:l + 1]), None,
                      ptr(self.tok_of_row[l]), ptr(self.piece_row[l]), ptr(self.piece_rows[l]),
                      ptr(self.exp_begin[l]), ptr(x), d, ptr(self.ws_ffn) if gather_fused else None,
                      ptr(self.ws_exec), self.ws_exec_n, sp)
            n = 1 + 3  # router | chunk prefixes, slot layout, ranks (+ permute)
        else:  # E > 128: split pre-pass + split-bf16 GEMM + recheck, then the four-kernel map
            _lib.call("mp_route_top1_ex", ptr(x), d, T, d, ptr(lay.w_hl), ptr(lay.w32), ptr(lay.w_abs), E, lay.Eg,
                      ptr(self.route[l]), ptr(self.ws_router), self.ws_router_n, sp)
            _lib.call("mp_exec_map", ptr(self.route[l]), 1, T, E, self.max_slots, split, ptr(self.res[l]),
                      ptr(self.exec_slot[l]), ptr(self.corrective[l]), ptr(self.exec_slots[l:l + 1]), None,
                      ptr(self.tok_of_row[l]), ptr(self.piece_row[l]), ptr(self.piece_rows[l]),
                      ptr(self.exp_begin[l]), ptr(self.ws_exec), self.ws_exec_n, sp)
            n = 3 + 4
            gather_fused = False
        if not gather_fused:
            _lib.call("mp_ffn_gather", ptr(x), T, d, F, E, ptr(self.tok_of_row[l]), ptr(self.ws_ffn), self.ws_ffn_n,
                      sp)
            n += 1
        if cfg.physical_replicas:  # materialise the layer's residency in the weight pool, then run on it
            E_, R, P = cfg.num_experts, self.pool_R, self.pool_P
            st = self.pool_state[l]
            _lib.call("mp_pool_update", ptr(self.res[l]), E_, R, P, ptr(st), sp)
            _lib.call("mp_replica_copy", ptr(lay.U), ptr(lay.V), ptr(self.pool_u[l]), ptr(self.pool_v[l]),
                      2 * d * F, P, ptr(st), E_, R, sp)
            _lib.call("mp_piece_pool", ptr(self.piece_row[l]), ptr(self.exp_begin[l]), E_, ptr(self.tok_of_row[l]),
                      ptr(self.exec_slot[l]), ptr(st), R, P, ptr(self.piece_wbase[l]), self.pstride, sp)
            n += 4  # pool update | copies (two passes) | piece -> slot
            if ev is not None:
                ev[0].record(sp)
            flags = lay.tiled
            _lib.call("mp_ffn_up_pool", T, d, F, E, P, ptr(self.pool_u[l]), flags, ptr(self.piece_row[l]),
                      ptr(self.piece_rows[l]), ptr(self.exp_begin[l]), ptr(self.piece_wbase[l]), ptr(self.ws_ffn),
                      self.ws_ffn_n, sp)
            if ev is not None:
                ev[1].record(sp)
            _lib.call("mp_ffn_down_pool", ptr(x), T, d, F, E, P, ptr(self.pool_v[l]), flags, ptr(self.tok_of_row[l]),
                      ptr(self.piece_row[l]), ptr(self.piece_rows[l]), ptr(self.exp_begin[l]),
                      ptr(self.piece_wbase[l]), ptr(self.ws_ffn), self.ws_ffn_n, sp)
            if ev is not None:
                ev[2].record(sp)
            return n + 2
        if ev is not None:
            ev[0].record(sp)
        flags = lay.tiled | (2 if use_pair else 0)
        _lib.call("mp_ffn_up", T, d, F, E, ptr(lay.U), flags, ptr(self.piece_row[l]), ptr(self.piece_rows[l]),
                  ptr(self.exp_begin[l]), ptr(self.ws_ffn), self.ws_ffn_n, sp)
        if ev is not None:
            ev[1].record(sp)
        _lib.call("mp_ffn_down", ptr(x), T, d, F, E, ptr(lay.V), flags, ptr(self.tok_of_row[l]),
                  ptr(self.piece_row[l]), ptr(self.piece_rows[l]), ptr(self.exp_begin[l]), ptr(self.ws_ffn),
                  self.ws_ffn_n, sp)
        if ev is not None:
            ev[2].record(sp)
        return n + 2

    # ------------------------------------------------------------------ expert parallelism
    def enable_expert_parallel(self, group=None, peer_cap: int | None = 0, cap_factor: float = 1.25,
                               p2p: bool = False) -> None:
        """Shard experts' work over the ranks of ``group`` (one process per GPU, NCCL):
        every rank keeps all weights, routes its own tokens and dispatches them to the GPU
        hosting their replica (paper_2605_11537_b200/ep.py). Residency is planned from the
        all-gathered predicted assignments so every rank holds the same state.

        ``peer_cap`` > 0: fixed-split dispatch with that many rows per (source, destination)
        block -- no host read-back, the step can be captured in a CUDA graph; ``None``:
        cap_factor x T / G rows rounded up to 128 (T at G = 1): the row-budgeted replica
        placement gives every GPU ~T rows, ~T / G from each source, so 25 % headroom covers
        statistically similar shards (a layer that needs more is re-run compactly); 0: compact
        dispatch (split sizes read back once per layer). The padding travels: the all-to-alls
        move G x peer_cap rows. ``p2p``: the fixed-split dispatch and combine over peer memory
        (NVLink P2P through CUDA IPC mappings, no all-to-all; ep.py)."""
        import torch.distributed as dist

        from .errors import ConfigurationError
        from .ep import CudaEpKernels, ExpertParallelMoE

        if self.cfg.physical_replicas:
            # every GPU keeps all master weights under EP: a replica hosted on a GPU
            # reads them there, so per-slot weight pools would only add copies
            raise ConfigurationError("physical replicas are a single-GPU mode; expert parallelism reads the "
                                     "resident master weights on every GPU")
        self.group = group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        cfg = self.cfg
        # slots of the global plan: G * C capacity slots + at most one corrective replica per expert
        if peer_cap is None:
            want = math.ceil(cap_factor * cfg.tokens / self.world / 128) * 128
            peer_cap = cfg.tokens if self.world == 1 else min(cfg.tokens, want)
        max_slots = self.world * cfg.capacity + cfg.num_experts
        k = CudaEpKernels(self.layers, cfg.tokens, self.world, self.rank, max_slots, peer_cap=peer_cap, p2p=p2p)
        if p2p:
            # map the peers, agree that every rank could, then check the mappings + device barrier
            # once and agree again; any problem on any rank -> every rank takes the all-to-all form
            # of the same fixed-split layout (each step below runs the same collectives on all ranks)
            def agree(ok: bool) -> bool:
                if self.world == 1:
                    return ok
                flag = torch.tensor([0 if ok else 1], dtype=torch.int32, device=self.dev)
                dist.all_reduce(flag, group=group)
                return int(flag.item()) == 0

            try:
                k.connect(group)
                ok = True
            except Exception:  # noqa: BLE001 -- a peer that cannot be mapped selects the NCCL path
                ok = False
            ok = agree(ok)
            if ok:
                try:
                    ok = k.verify_peers()
                except Exception:  # noqa: BLE001
                    ok = False
                ok = agree(ok)
            if not ok:
                k = CudaEpKernels(self.layers, cfg.tokens, self.world, self.rank, max_slots, peer_cap=peer_cap)
        self.ep_p2p = bool(getattr(k, "p2p", False))
        self.ep = ExpertParallelMoE(k, cfg.num_layers, cfg.num_experts, group)
        self.ep.res = self.res  # one residency state for placement and execution
        GT = self.world * cfg.tokens
        i32 = dict(dtype=torch.int32, device=self.dev)
        self.g_assign = torch.empty(cfg.num_layers, GT, **i32)
        self.g_slot = torch.empty(cfg.num_layers, GT, **i32)
        self.g_event = torch.empty(cfg.num_layers, GT, **i32)
        self.ws_gplace_n = _lib.size_query("mp_place_workspace_bytes", cfg.num_layers, GT, cfg.num_experts)
        self.ws_gplace = torch.empty(self.ws_gplace_n, dtype=torch.uint8, device=self.dev)
        self.ws_ghist_n = _lib.size_query("mp_histogram_workspace_bytes", cfg.num_layers, GT, cfg.num_experts)
        self.ws_ghist = torch.empty(self.ws_ghist_n, dtype=torch.uint8, device=self.dev)
        if self.ep_p2p and self.world > 1:
            # the step's other all-gathers over peer memory too: the predicted assignments (once per
            # step) and the sharded SRU's carry maps (per SRU layer; two buffers by layer parity, so a
            # rank running ahead never overwrites maps a slower rank has not folded yet)
            d = self.dp
            self.sru_tots_pp = torch.zeros(2, self.world, 2 * d, device=self.dev)
            self.t_sru_tots = [k._mem.table(self.sru_tots_pp[0]), k._mem.table(self.sru_tots_pp[1])]
            self.t_g_assign = k._mem.table(self.g_assign)
        # tests: issue the collectives (NCCL all-gathers, all-to-alls) even when world == 1
        self.force_collectives = False

    def predict_sharded(self, x: torch.Tensor, sp: int) -> int:
        """Predictor over a token-sharded batch: the G ranks' token ranges are ONE sequence
        (the reference scans the whole batch, src/predictor.py:175-195). Per SRU layer each
        rank projects its rows, reduces its range to one affine carry map (2d fp32),
        all-gathers the maps, folds the lower ranks' maps into its carry-in and replays
        from it."""
        import torch.distributed as dist

        cfg, T, d = self.cfg, self.cfg.tokens, self.dp
        if getattr(self, "sru_tot", None) is None:
            self.sru_tot = torch.empty(2 * d, device=self.dev)
            self.sru_tots = torch.empty(self.world, 2 * d, device=self.dev)
            self.sru_carry_in = torch.empty(d, device=self.dev)
        _lib.call("mp_f32_to_bf16", ptr(x), ptr(self.x16), T * d, sp)
        n = 1
        cur32, cur16 = x, self.x16
        for i, (W, B) in enumerate(zip(self.sru.w_cat, self.sru.b_cat)):
            h32, h16 = self.h32[i % 2], self.h16[i % 2]
            _lib.call("mp_sru_project", ptr(cur16), ptr(W), ptr(B), T, d, ptr(self.ws_sru), self.ws_sru_n, sp)
            _lib.call("mp_sru_scan_total", T, d, ptr(self.sru_tot), ptr(self.ws_sru), self.ws_sru_n, sp)
            if getattr(self, "ep_p2p", False) and self.world > 1:  # peer stores + device barrier
                tots = self.sru_tots_pp[i % 2]
                _lib.call("mp_peer_allgather_i32", ptr(self.sru_tot), 1, 2 * d, self.rank, self.world,
                          ptr(self.t_sru_tots[i % 2]), 0, sp)
                self.ep.k.barrier()
            else:
                tots = self.sru_tots
                parts = list(self.sru_tots.unbind(0))
                dist.all_gather(parts, self.sru_tot, group=self.group)
            _lib.call("mp_sru_fold_carry", ptr(tots), self.rank, d, None, ptr(self.sru_carry_in), sp)
            _lib.call("mp_sru_scan_finish", ptr(cur32), T, d, ptr(self.sru_carry_in), ptr(h32), ptr(h16), None,
                      ptr(self.nonfinite), ptr(self.ws_sru), self.ws_sru_n, sp)
            n += 6  # GEMM | aggregate, carry | fold | carry, replay
            cur32, cur16 = h32, h16
        _lib.call("mp_heads_argmax", ptr(cur16), ptr(self.sru.heads), T, d, cfg.num_layers, cfg.num_experts,
                  self.sru.Eg, ptr(self.assign), sp)
        return n + 1

    def step_ep(self, x: torch.Tensor, events=None) -> int:
        """One expert-parallel step. Fixed-split dispatch (``peer_cap``): outside a CUDA-graph
        capture the overflow flag is checked once at the end; on overflow the step is rolled
        back (input stream and residency state) and re-run with compact dispatch. A captured
        step leaves the check to the caller (``ep_overflowed``)."""
        k = self.ep.k
        if not k.peer_cap or torch.cuda.is_current_stream_capturing():
            return self._step_ep(x, events)
        if k.p2p:
            self.check_peer_barriers()
        x0, res0 = x.clone(), self.res.clone()
        k.overflow.zero_()
        n = self._step_ep(x, events)
        if k.p2p:
            self.check_peer_barriers()
        if int(k.overflow.item()):
            x.copy_(x0)
            self.res.copy_(res0)
            cap, k.peer_cap = k.peer_cap, 0
            try:
                n = self._step_ep(x, events)
            finally:
                k.peer_cap = cap
                k.overflow.zero_()
        return n

    def check_peer_barriers(self) -> None:
        """Peer-memory EP: raise if a device barrier since the last check gave up waiting for a
        rank (5 s); the steps since then are invalid."""
        from .errors import DeviceError

        k = self.ep.k
        if getattr(k, "p2p", False) and int(k.peer_err.item()):
            k.peer_err.zero_()
            raise DeviceError("peer-memory expert parallelism: a device barrier timed out waiting for a rank")

    def ep_overflowed(self) -> bool:
        """Fixed-split dispatch: did any layer since the last reset need more than peer_cap rows
        for some peer (that layer did nothing; the step must be re-run)? Resets the flag."""
        k = self.ep.k
        hit = bool(int(k.overflow.item()))
        k.overflow.zero_()
        return hit

    def _step_ep(self, x: torch.Tensor, events=None) -> int:
        import torch.distributed as dist

        cfg, L, T, E = self.cfg, self.cfg.num_layers, self.cfg.tokens, self.cfg.num_experts
        sp = stream_ptr()
        coll = self.world > 1 or self.force_collectives
        self.ep.force_collectives = self.force_collectives
        n = self.predict_sharded(x, sp) if coll else self.predict(x, sp)
        parts = list(self.g_assign.view(L, self.world, T).unbind(1))
        if coll and getattr(self, "ep_p2p", False) and self.world > 1:  # peer stores + device barrier
            _lib.call("mp_peer_allgather_i32", ptr(self.assign), L, T, self.rank, self.world, ptr(self.t_g_assign),
                      self.world * T, sp)
            self.ep.k.barrier()
        elif coll:
            gathered = [torch.empty(L, T, dtype=torch.int32, device=self.dev) for _ in range(self.world)]
            dist.all_gather(gathered, self.assign, group=self.group)
            for r in range(self.world):
                parts[r].copy_(gathered[r])
        else:
            self.g_assign.copy_(self.assign)
        GT = self.world * T
        unit = DISTINCT_ONLY_UNIT if cfg.replication == "off" else cfg.demand_unit
        _lib.call("mp_histogram_ws", ptr(self.g_assign), L, GT, E, ptr(self.demand), ptr(self.ws_ghist),
                  self.ws_ghist_n, sp)
        cap = cfg.capacity * self.world  # global capacity G * C_g
        _lib.call("mp_cap_replicas", ptr(self.demand), L, E, cap, unit, ptr(self.caps), ptr(self.infeasible), sp)
        _lib.call("mp_place", ptr(self.g_assign), L, GT, E, ptr(self.caps), cap, cap, ptr(self.res), ptr(self.g_slot),
                  ptr(self.g_event), ptr(self.offloads), ptr(self.fallback), ptr(self.num_slots), ptr(self.ws_gplace),
                  self.ws_gplace_n, sp)
        for l in range(L):
            self.ep.layer(l, x, events[l] if events is not None else None)
        return n + 7 + L * 12

    def step(self, x: torch.Tensor, events=None) -> int:
        """Run one batch on the current stream; x (T, d) fp32 is the residual stream (in/out).

        events: optional list (per layer) of 3 CUDA events bracketing GEMM1 / GEMM2.
        Returns the number of kernel launches issued."""
        if getattr(self, "ep", None) is not None:
            return self.step_ep(x, events)
        sp = stream_ptr()
        n = self.predict(x, sp)
        n += self.plan_and_place(sp)
        for l in range(self.cfg.num_layers):
            n += self.layer(l, x, sp, events[l] if events is not None else None)
        self.launches_per_step = n
        return n

    def step_checked(self, x: torch.Tensor, rows: torch.Tensor) -> list[torch.Tensor]:
        """Eager single-device step that also snapshots the residual-stream rows ``rows`` before
        every MoE layer and after the last one (L + 1 tensors), for correctness checks taken
        outside any timed region (bench.py, tests)."""
        sp = stream_ptr()
        self.predict(x, sp)
        self.plan_and_place(sp)
        snaps = []
        for l in range(self.cfg.num_layers):
            snaps.append(x[rows].clone())
            self.layer(l, x, sp)
        snaps.append(x[rows].clone())
        return snaps

    def expert_weights_untiled(self, l: int, e: int) -> tuple[torch.Tensor, torch.Tensor]:
        """(U_e (F, d), V_e (d, F)) bf16 of layer l, expert e, back in the reference layout
        (router_oracle.py:26-27) from the pre-tiled device copy."""
        lay = self.layers[l]
        d, F = lay.dp, lay.Fp
        ubn = lay.ubn
        u = lay.U.view(lay.E, F // ubn, d // 64, ubn, 64)[e].permute(0, 2, 1, 3).reshape(F, d)
        v = lay.V.view(lay.E, d // lay.vbn, F // 64, lay.vbn, 64)[e].permute(0, 2, 1, 3).reshape(d, F)
        return u, v

    def toy_params(self):
        """The engine's MoE weights as the reference's ToyMoeParams (float32 numpy, reference
        layouts; bf16 values, so the drop-in API re-quantises them losslessly)."""
        import numpy as np

        from .router_oracle import ToyMoeParams

        cfg, L, E, d, F = self.cfg, self.cfg.num_layers, self.cfg.num_experts, self.dp, self.Fp
        router = np.stack([self.wl.router(l).cpu().numpy() for l in range(L)])
        u = np.empty((L, E, F, d), dtype=np.float32)
        v = np.empty((L, E, d, F), dtype=np.float32)
        for l in range(L):
            lay = self.layers[l]
            u[l] = lay.U.view(E, F // lay.ubn, d // 64, lay.ubn, 64).permute(0, 1, 3, 2, 4).reshape(E, F, d) \
                .float().cpu().numpy()
            v[l] = lay.V.view(E, d // lay.vbn, F // 64, lay.vbn, 64).permute(0, 1, 3, 2, 4).reshape(E, d, F) \
                .float().cpu().numpy()
        return ToyMoeParams(router, u, v)

    def sru_params(self):
        """The engine's predictor as the reference's SruParams (float64 host copies)."""
        from .predictor import SruLayerParams, SruParams

        return SruParams(layers=[SruLayerParams(*lay) for lay in self.sru_host], heads=self.heads_host)

    # ------------------------------------------------------------------ CUDA graph
    def capture(self, x: torch.Tensor, events=None) -> "StepGraph":
        """Capture one step over the fixed residual-stream buffer ``x`` (run ``step`` once
        first so every kernel attribute is configured). Replays need no host work."""
        sp = stream_ptr()
        _lib.call("mp_graph_begin", sp)
        try:
            n = self.step(x, events)
        except Exception:
            ex = ctypes.c_void_p()
            _lib.load_library().mp_graph_end(sp, ctypes.byref(ex))
            raise
        return _end_capture(sp, n)

    def capture_call(self, fn) -> "StepGraph":
        """Capture ``fn(sp) -> launches`` on the current stream into a replayable graph."""
        sp = stream_ptr()
        _lib.call("mp_graph_begin", sp)
        try:
            n = fn(sp)
        except Exception:
            ex = ctypes.c_void_p()
            _lib.load_library().mp_graph_end(sp, ctypes.byref(ex))
            raise
        return _end_capture(sp, n)

    def consume(self, x: torch.Tensor, sp: int, events=None) -> int:
        """Consumer half of a step: plan + place the predicted table, then the MoE layers."""
        n = self.plan_and_place(sp)
        for l in range(self.cfg.num_layers):
            n += self.layer(l, x, sp, events[l] if events is not None else None)
        return n

    # ------------------------------------------------------------------ accounting
    def expert_weight_bytes(self) -> int:
        """bf16 bytes of one expert's U + V (4 d F)."""
        return 4 * self.cfg.d_model * self.cfg.d_ff

    def touched_experts(self) -> torch.Tensor:
        """(L,) experts that received tokens in the last step (device)."""
        return (self.exp_begin[:, 1:] > self.exp_begin[:, :-1]).sum(dim=1)

    def layer_counts(self):
        """(L, 5) device counts of the last step -- {LOAD (placement + corrective), REPLICATE,
        OFFLOAD events, longest replica-slot queue, slots} (csrc/counts.cu)."""
        from .simulator import layer_counts

        return layer_counts(self.exec_slot, self.exec_slots, self.max_slots, token_event=self.pred_event,
                            offloads=self.offloads, corrective=self.corrective)

    def metrics(self, cost=None, layer_latency=None):
        """The reference's per-batch ``Metrics`` (src/simulator.py:210-235) of the last step from
        its device counts; ``layer_latency`` (per MoE layer, e.g. measured ms) replaces the
        cost model's layer makespans. Returns (Metrics, counts)."""
        from .simulator import CostModel, metrics_from_counts

        counts = self.layer_counts()
        acc = float((self.assign == self.route).float().mean().item())
        return metrics_from_counts(counts, self.cfg.tokens, cost or CostModel(), acc, layer_latency), counts


class OverlappedPipeline:
    """The paper's two-actor schedule (Alg. 1 + Alg. 2; reference src/pipeline.py:70-139)
    on two CUDA streams instead of a producer thread and a FIFO: the hash-table builder
    (SRU predictor + heads) for batch i+1 runs on its own stream while batch i is planned,
    placed and forwarded; double-buffered inputs/assignments, events in place of the queue
    (queue capacity 1, the reference default src/pipeline.py:35-45). Each half is one
    CUDA graph. Planning/placement stay in batch order on the consumer stream, so results
    are identical to the sequential schedule (the reference's mode_equivalence_check)."""

    def __init__(self, pipe: "MoEPipeline", events=None, ffn_sms: int = 0, predictor_sms: int = 0):
        """ffn_sms / predictor_sms: persistent grids of the expert GEMMs and of the predictor
        GEMMs (mp_set_sm_partition) so both halves find free SMs; 0 = all SMs. The consumer
        (MoE layers) stream has the higher priority."""
        self.pipe = pipe
        T, d = pipe.cfg.tokens, pipe.dp
        dev = pipe.dev
        self.xbuf = [torch.empty(T, d, device=dev) for _ in range(2)]
        self.assign = [pipe.assign, torch.empty_like(pipe.assign)]
        self.sp, self.sf = torch.cuda.Stream(priority=0), torch.cuda.Stream(priority=-1)
        _lib.call("mp_set_sm_partition", int(ffn_sms), int(predictor_sms))
        self.pred_ev = [torch.cuda.Event() for _ in range(2)]
        self.cons_ev = [torch.cuda.Event() for _ in range(2)]
        self.g_pred, self.g_cons = [], []
        for j in range(2):  # warm (configures kernel attributes) then capture each half per slot
            pipe.assign = self.assign[j]
            with torch.cuda.stream(self.sp):
                pipe.predict(self.xbuf[j], stream_ptr())
                self.g_pred.append(pipe.capture_call(lambda sp, j=j: pipe.predict(self.xbuf[j], sp)))
            with torch.cuda.stream(self.sf):
                self.g_cons.append(pipe.capture_call(lambda sp, j=j: pipe.consume(self.xbuf[j], sp, events)))
        pipe.assign = self.assign[0]
        torch.cuda.synchronize()
        _lib.call("mp_set_sm_partition", 0, 0)  # the captured graphs keep their grids
        self.launches = self.g_pred[0].launches + self.g_cons[0].launches

    def run(self, batches, n: int, timer=None) -> None:
        """Process ``n`` batches (cycled from ``batches`` (T, d) device tensors)."""
        for i in range(n + 1):
            if i < n:  # producer: batch i
                j = i % 2
                with torch.cuda.stream(self.sp):
                    if i >= 2:
                        self.sp.wait_event(self.cons_ev[j])
                    elif i == 0 and timer is not None:
                        timer[0].record(self.sp)
                    self.xbuf[j].copy_(batches[i % len(batches)])
                    self.g_pred[j].replay()
                    self.pred_ev[j].record(self.sp)
            if i >= 1:  # consumer: batch i - 1
                j = (i - 1) % 2
                with torch.cuda.stream(self.sf):
                    self.sf.wait_event(self.pred_ev[j])
                    self.g_cons[j].replay()
                    self.cons_ev[j].record(self.sf)
        if timer is not None:
            with torch.cuda.stream(self.sf):
                timer[1].record(self.sf)


class DeviceEvent:
    """CUDA event owned by libmoempmc (valid inside captured graphs)."""

    def __init__(self):
        self.h = ctypes.c_void_p()
        _lib.call("mp_event_create", ctypes.byref(self.h))

    def record(self, sp: int):
        _lib.call("mp_event_record", self.h, sp)

    def elapsed_ms(self, end: "DeviceEvent") -> float:
        ms = ctypes.c_float()
        _lib.call("mp_event_elapsed_ms", self.h, end.h, ctypes.byref(ms))
        return float(ms.value)

    def __del__(self):
        try:
            if self.h:
                _lib.load_library().mp_event_destroy(self.h)
        except Exception:
            pass


def _end_capture(sp: int, issued: int) -> "StepGraph":
    """End a capture; the graph's own kernel-node count is the launches per replay (the
    host-side tally ``issued`` must agree -- a mismatch means a stale count)."""
    ex, k = ctypes.c_void_p(), ctypes.c_int32(0)
    _lib.call("mp_graph_end_counted", sp, ctypes.byref(ex), ctypes.byref(k))
    g = StepGraph(ex, int(k.value))
    g.issued = issued
    return g


class StepGraph:
    def __init__(self, exec_handle: ctypes.c_void_p, launches: int):
        self.h = exec_handle
        self.launches = launches

    def replay(self):
        _lib.call("mp_graph_launch", self.h, stream_ptr())

    def destroy(self):
        """Release the executable graph now (a graph holding captured NCCL collectives must be
        destroyed before its process group)."""
        try:
            if self.h:
                _lib.load_library().mp_graph_destroy(self.h)
        except Exception:
            pass
        self.h = None

    def __del__(self):
        self.destroy()


def _layer_from_device(router: torch.Tensor, u: torch.Tensor, v: torch.Tensor, ffn: str = "two") -> DeviceMoeLayer:
    """DeviceMoeLayer from device tensors already in kernel layout (d % 64 == 0, F % 256 == 0)."""
    lay = DeviceMoeLayer.__new__(DeviceMoeLayer)
    E, d = router.shape
    F = u.shape[1]
    lay.E, lay.d, lay.F, lay.dp, lay.Fp = E, d, F, d, F
    lay.Eg = router_eg(E)
    w32 = router.float().contiguous()
    hi = w32.to(torch.bfloat16)
    lo = (w32 - hi.float()).to(torch.bfloat16)
    lay.w_hl = torch.zeros(lay.Eg, 2 * d, device=router.device, dtype=torch.bfloat16)
    lay.w_hl[:E, :d] = hi
    lay.w_hl[:E, d:] = lo
    lay.w32 = w32
    lay.w_abs = torch.empty(d, device=router.device)
    _lib.call("mp_router_weight_absmax", ptr(w32), E, d, ptr(lay.w_abs), stream_ptr())
    # pre-tiled B operands: each TMA box of the grouped GEMMs is one contiguous 32 KB burst
    u2, v2 = u.reshape(E * F, d).contiguous(), v.reshape(E * d, F).contiguous()
    lay.U, lay.V = torch.empty_like(u2), torch.empty_like(v2)
    ubn = _lib.size_query("mp_ffn_up_bn", F)
    vbn = 256 if ffn == "pair" else _lib.size_query("mp_ffn_down_bn", d)  # the CTA-pair kernels read BN 256
    _lib.call("mp_tile_kmajor", ptr(u2), ptr(lay.U), E, F, d, ubn, stream_ptr())
    _lib.call("mp_tile_kmajor", ptr(v2), ptr(lay.V), E, d, F, vbn, stream_ptr())
    lay.tiled = 1
    lay.ubn, lay.vbn = ubn, vbn
    lay.ffn = ffn
    del u2, v2
    return lay


DeviceMoeLayer.from_device = staticmethod(_layer_from_device)
