"""Expert-parallel MoE forward over G ranks (one process per GPU, NCCL), SURVEY.md §8(e).

Tokens are sharded contiguously by position; every GPU holds all expert weights
(14.5 GB at Switch-base-128 -- far inside 180 GB of HBM), so "placing" a
replica only decides which GPU *reads* that expert's weights and computes its
tokens. Per MoE layer, on every rank:

  1. route the local tokens                      (mp_route_top1_ex)
  2. local expert counts -> all-gather C (G x E)  (mp_histogram_ws + all_gather)
  3. plan (identical on all ranks): residency + corrective replicas, global
     stable ranks, the slot list cut into G blocks of equal rows (slot -> GPU),
     per-peer row counts,
     send positions, local replica pieces         (mp_ep_plan)
  4. dispatch: pack bf16 rows by destination, variable all-to-all
  5. receiver: rows to slot-major global-token order (mp_ep_recv_layout,
     mp_gather_rows_bf16), grouped expert GEMMs whose GEMM2 epilogue writes the
     fp32 results straight into receive order (mp_ffn_up/down)
  6. combine: reverse all-to-all, x[t] += y[send_pos[t]]  (mp_ep_combine)

Because the global ranks, slots, rows and per-row arithmetic are those of the
single-device path, the output is bit-identical to one GPU running the whole
batch. In the compact mode the all-to-all byte counts are data dependent, so each layer
does one small device->host read of the split sizes. In the fixed-split mode
(``peer_cap`` > 0) every (source, destination) block of the send / receive buffers has
peer_cap rows: the all-to-alls have static equal splits, nothing reaches the host and the
whole step can be captured in one CUDA graph; a layer that would need more than peer_cap
rows for some peer sets an overflow flag and does nothing, and the caller re-runs the step
in the compact mode (MoEPipeline.step does so, checking the flag once per step).

Peer-memory mode (``p2p``, fixed splits): no all-to-all at all. Every rank maps the other
ranks' receive buffers, receive-token arrays, barrier flags and residual streams into its
address space once (CUDA IPC, NVLink P2P on NVSwitch); per layer the source writes its rows
straight into the destination's receive block (``mp_ep_pack_peer``), a device barrier
(``mp_peer_barrier``) hands them over, and the destination's GEMM2 epilogue ADDS each result
row into the home rank's residual stream over NVLink (``mp_ffn_down_peer``: the combine fused
into the GEMM), followed by a second barrier. Same bits as the all-to-all form.

The kernel layer is pluggable: ``CudaEpKernels`` (the product) or, in the
CPU multi-process tests only, a numpy restatement from ``oracle/``.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from . import _lib
from ._dev import ptr, stream_ptr
from .errors import ConfigurationError
from .router_oracle import DeviceMoeLayer, route_device


@dataclass
class EpPlan:
    send_counts: list[int]
    recv_counts: list[int]
    n_local: int
    send_pos: torch.Tensor
    piece_row: torch.Tensor
    piece_rows: torch.Tensor
    exp_begin: torch.Tensor


class PeerMemory:
    """Peer address tables of same-role buffers over a process group: torch's CUDA IPC
    (``UntypedStorage._share_cuda_`` / ``_new_shared_cuda``, i.e. cudaIpcGetMemHandle /
    cudaIpcOpenMemHandle) exchanged with ``all_gather_object``; entry ``rank`` is the local
    pointer. The mapped storages are kept alive with this object."""

    def __init__(self, group, world: int, rank: int, dev):
        self.group, self.world, self.rank, self.dev = group, world, rank, dev
        self._keep = []
        self.failed = False  # a peer mapping could not be made here (the collectives still ran)

    def table(self, t: torch.Tensor) -> torch.Tensor:
        """int64 device array: entry g = address of rank g's tensor in the same role as ``t``
        (collective over the group: every rank calls it with its own tensor)."""
        ptrs = [t.data_ptr()] * self.world
        if self.world > 1:
            off = t.storage_offset() * t.element_size()
            objs = [None] * self.world
            dist.all_gather_object(objs, (t.untyped_storage()._share_cuda_(), off), group=self.group)
            for g, (handle, og) in enumerate(objs):
                if g != self.rank:
                    # kernels on this device dereference the peer's memory: peer access first. A
                    # failure is recorded, not raised, so every rank still takes part in the
                    # remaining exchanges; the caller checks ``failed`` with the other ranks.
                    try:
                        _lib.call("mp_enable_peer_access", int(handle[0]))
                        st = torch.UntypedStorage._new_shared_cuda(*handle)
                        self._keep.append(st)
                        ptrs[g] = st.data_ptr() + og
                    except Exception:  # noqa: BLE001
                        self.failed = True
                        ptrs[g] = 0
        return torch.tensor(ptrs, dtype=torch.int64, device=self.dev)


class CudaEpKernels:
    """Device implementation (libmoempmc.so) of the per-rank EP steps."""

    dispatch_dtype = torch.bfloat16

    def __init__(self, layers: list[DeviceMoeLayer], tokens: int, world: int, rank: int, max_slots: int,
                 peer_cap: int = 0, p2p: bool = False):
        self.layers = layers
        self.T, self.G, self.rank, self.max_slots = tokens, world, rank, max_slots
        self.peer_cap = int(peer_cap)  # rows per (source, destination) block; 0: compact, sizes read back
        lay = layers[0]
        self.E, self.d, self.F = lay.E, lay.dp, lay.Fp
        dev = lay.U.device
        self.dev = dev
        i32 = dict(dtype=torch.int32, device=dev)
        self.pstride = max_slots + (world * tokens + 127) // 128
        self.cap_rows = world * tokens  # worst case: every token of every rank lands here
        self.ws_n = _lib.size_query("mp_ep_workspace_bytes", world, tokens, self.E, max_slots)
        self.ws = torch.empty(self.ws_n, dtype=torch.uint8, device=dev)
        self.hist_n = _lib.size_query("mp_histogram_workspace_bytes", 1, tokens, self.E)
        self.hist_ws = torch.empty(max(self.hist_n, 256), dtype=torch.uint8, device=dev)
        self.ffn_n = _lib.size_query("mp_ffn_workspace_bytes", self.cap_rows, self.d, self.F)
        self.ffn_ws = torch.empty(self.ffn_n, dtype=torch.uint8, device=dev)
        self.counts_buf = torch.empty(self.E, **i32)
        self.sizes = torch.empty(2 * world + 1, **i32)  # send counts | recv counts | local rows
        self.sc, self.rc, self.nloc = self.sizes[:world], self.sizes[world:2 * world], self.sizes[2 * world:]
        self.sizes_host = torch.empty(2 * world + 1, dtype=torch.int32, pin_memory=True)
        self.sizes_ready = torch.cuda.Event()
        # capacity buffers (no per-layer allocation): a rank sends at most T rows and receives
        # at most G * T
        self.overflow = torch.zeros(1, **i32)  # fixed-split mode: some layer needed more than peer_cap rows
        send_rows = max(tokens, world * self.peer_cap)
        self.sendbuf = torch.empty(send_rows, self.d, dtype=torch.bfloat16, device=dev)
        self.recvbuf = torch.empty(self.cap_rows, self.d, dtype=torch.bfloat16, device=dev)
        self.ybuf = torch.empty(self.cap_rows, self.d, dtype=torch.float32, device=dev)
        self.yback = torch.empty(send_rows, self.d, dtype=torch.float32, device=dev)
        self._packed_for = None
        # zero-filled: if a plan overflows max_slots its send positions are left untouched, and the
        # pack issued before the host sees the error must still write inside the send buffer
        self.send_pos = torch.zeros(tokens, **i32)
        self.piece_row = torch.empty(self.pstride, **i32)
        self.piece_rows = torch.empty(self.pstride, **i32)
        self.exp_begin = torch.empty(self.E + 1, **i32)
        self.recv_of_local = torch.zeros(self.cap_rows, **i32)
        # peer-memory mode: receive-token indices (peer-written), barrier flags + epoch, the
        # destination code of every local row; the peer tables are set by connect() / set_peers()
        self.p2p = bool(p2p)
        if self.p2p:
            if self.peer_cap <= 0:
                raise ConfigurationError("peer-memory expert parallelism needs the fixed-split layout (peer_cap > 0)")
            self.recv_tok = torch.zeros(world * self.peer_cap, **i32)
            self.flags = torch.zeros(world, **i32)
            self.epoch = torch.zeros(1, **i32)
            self.peer_err = torch.zeros(1, **i32)  # a barrier timed out (a rank never arrived)
            self.dst_of_row = torch.zeros(self.cap_rows, **i32)
            self.C_all = torch.zeros(world, self.E, **i32)  # every rank's expert counts (peer-written)
            self.t_recv = self.t_tok = self.t_flags = self.t_x = self.t_C = None
            self._x_ptr = None
            self._mem = None

    # ---------------------------------------------------------------- peer-memory mode
    def connect(self, group) -> None:
        """Map the peers' receive buffers, receive-token arrays and flags (collective)."""
        self._mem = PeerMemory(group, self.G, self.rank, self.dev)
        self.set_peers(self._mem.table(self.recvbuf), self._mem.table(self.recv_tok), self._mem.table(self.flags),
                       self._mem.table(self.C_all))
        if self._mem.failed:
            raise ConfigurationError("peer memory: a peer's buffers could not be mapped on this GPU")

    def verify_peers(self) -> bool:
        """Check the peer mappings and the device barrier once (collective): every rank stores a
        row and its index into every peer's receive block through the tables, a device barrier
        hands them over, and each rank checks what its peers wrote. False (on every rank that
        sees a problem) means: use the all-to-all path."""
        G, pc, d = self.G, self.peer_cap, self.d
        i32 = dict(dtype=torch.int32, device=self.dev)
        x = torch.full((G, d), float(self.rank + 1), device=self.dev)
        send_pos = torch.arange(G, **i32) * pc  # token g -> rank g, row rank * peer_cap
        self.recv_tok.fill_(-1)
        torch.cuda.synchronize()
        if G > 1:
            dist.barrier(group=self._mem.group)
        _lib.call("mp_ep_pack_peer", ptr(x), G, d, ptr(send_pos), pc, self.rank, ptr(self.t_recv), ptr(self.t_tok),
                  stream_ptr())
        self.barrier()
        torch.cuda.synchronize()
        rows = torch.arange(G, device=self.dev) * pc
        ok = int(self.peer_err.item()) == 0
        ok = ok and bool((self.recv_tok[rows] == self.rank).all().item())
        want = (torch.arange(G, device=self.dev, dtype=torch.float32) + 1).to(torch.bfloat16)
        ok = ok and bool(torch.equal(self.recvbuf[rows, 0], want))
        self.peer_err.zero_()
        return ok

    def set_peers(self, t_recv: torch.Tensor, t_tok: torch.Tensor, t_flags: torch.Tensor,
                  t_C: torch.Tensor = None) -> None:
        self.t_recv, self.t_tok, self.t_flags, self.t_C = t_recv, t_tok, t_flags, t_C

    def allgather_counts_peer(self, counts: torch.Tensor, barrier: bool = True) -> torch.Tensor:
        """Every rank's expert counts (G x E) by peer stores + a device barrier (no NCCL)."""
        _lib.call("mp_peer_allgather_i32", ptr(counts), 1, self.E, self.rank, self.G, ptr(self.t_C), 0, stream_ptr())
        if barrier:
            self.barrier()
        return self.C_all

    def register_stream(self, x: torch.Tensor, t_x: torch.Tensor = None) -> None:
        """Map every rank's residual stream (collective when the buffer changes; ``t_x`` given:
        a table built by the caller, e.g. a simulated job on one device)."""
        if t_x is not None:
            self.t_x, self._x_ptr = t_x, x.data_ptr()
        elif self._x_ptr != x.data_ptr():
            if torch.cuda.is_current_stream_capturing():
                raise ConfigurationError("peer-memory expert parallelism: run one eager step on this stream buffer "
                                         "before capturing (its peer mapping is a collective)")
            self.t_x, self._x_ptr = self._mem.table(x), x.data_ptr()

    def barrier(self) -> None:
        _lib.call("mp_peer_barrier", ptr(self.t_flags), self.rank, self.G, ptr(self.epoch), ptr(self.peer_err),
                  stream_ptr())

    def dispatch_peer(self, x: torch.Tensor, plan: EpPlan) -> None:
        """Rows straight into the destinations' receive blocks (peer stores); no barrier."""
        _lib.call("mp_ep_pack_peer", ptr(x), x.shape[0], self.d, ptr(plan.send_pos), self.peer_cap, self.rank,
                  ptr(self.t_recv), ptr(self.t_tok), stream_ptr())

    def expert_ffn_peer(self, plan: EpPlan, l: int, ev=None) -> None:
        """Grouped GEMMs on the received rows; GEMM2 adds every result row into its home rank's
        stream (peer reductions); no barrier."""
        n = self.G * self.peer_cap
        lay = self.layers[l]
        sp = stream_ptr()
        if not getattr(self, "_layout_ready", False):
            _lib.call("mp_ep_recv_layout", self.G, self.T, self.E, self.rank, self.max_slots, None,
                      ptr(self.recv_of_local), ptr(self.ws), self.ws_n, sp)
        self._layout_ready = False
        _lib.call("mp_ep_gather_peer", ptr(self.recvbuf), n, self.d, ptr(self.recv_of_local), ptr(self.nloc),
                  ptr(self.recv_tok), self.peer_cap, self.T, ptr(self.dst_of_row), ptr(self.ffn_ws), sp)
        if ev is not None:
            ev[0].record(sp)
        vflag = 64 if lay.tiled and getattr(lay, "vbn", 0) == 256 else 0
        _lib.call("mp_ffn_up", n, self.d, self.F, self.E, ptr(lay.U), lay.tiled, ptr(plan.piece_row),
                  ptr(plan.piece_rows), ptr(plan.exp_begin), ptr(self.ffn_ws), self.ffn_n, sp)
        if ev is not None:
            ev[1].record(sp)
        _lib.call("mp_ffn_down_peer", ptr(self.t_x), self.T, n, self.d, self.F, self.E, ptr(lay.V),
                  lay.tiled | vflag, ptr(self.dst_of_row), ptr(plan.piece_row), ptr(plan.piece_rows),
                  ptr(plan.exp_begin), ptr(self.ffn_ws), self.ffn_n, sp)
        if ev is not None:
            ev[2].record(sp)

    def route(self, x: torch.Tensor, l: int) -> torch.Tensor:
        return route_device(x, self.layers[l])

    def counts(self, route: torch.Tensor) -> torch.Tensor:
        _lib.call("mp_histogram_ws", ptr(route), 1, route.shape[0], self.E, ptr(self.counts_buf), ptr(self.hist_ws),
                  self.hist_n, stream_ptr())
        return self.counts_buf

    def plan(self, route: torch.Tensor, C: torch.Tensor, res: torch.Tensor, x: torch.Tensor = None) -> EpPlan:
        """Plan the layer; the split sizes come back to the host (one small D2H per layer: NCCL's
        variable all-to-all needs them). With ``x`` the dispatch rows are packed into the
        capacity send buffer BEFORE the host waits, so the pack overlaps the read-back."""
        T = route.shape[0]
        sp = stream_ptr()
        if self.peer_cap:  # fixed splits: no host read-back, graph-capturable
            _lib.call("mp_ep_plan_cap", ptr(route), T, ptr(C), self.G, self.E, self.rank, self.max_slots, 1,
                      self.peer_cap, ptr(self.overflow), ptr(res), ptr(self.sc), ptr(self.rc), ptr(self.nloc),
                      ptr(self.send_pos), ptr(self.piece_row), ptr(self.piece_rows), ptr(self.exp_begin),
                      ptr(self.ws), self.ws_n, sp)
            n = self.G * self.peer_cap
            if x is not None:
                _lib.call("mp_ep_pack", ptr(x), T, self.d, ptr(self.send_pos), ptr(self.sendbuf), sp)
            _lib.call("mp_ep_recv_layout", self.G, self.T, self.E, self.rank, self.max_slots, None,
                      ptr(self.recv_of_local), ptr(self.ws), self.ws_n, sp)
            self._packed_for = x
            self._layout_ready = True
            return EpPlan([self.peer_cap] * self.G, [self.peer_cap] * self.G, n, self.send_pos[:T], self.piece_row,
                          self.piece_rows, self.exp_begin)
        _lib.call("mp_ep_plan", ptr(route), T, ptr(C), self.G, self.E, self.rank, self.max_slots, 1, ptr(res),
                  ptr(self.sc), ptr(self.rc), ptr(self.nloc), ptr(self.send_pos), ptr(self.piece_row),
                  ptr(self.piece_rows), ptr(self.exp_begin), ptr(self.ws), self.ws_n, sp)
        self.sizes_host.copy_(self.sizes, non_blocking=True)
        self.sizes_ready.record()
        self._packed_for = None
        self._layout_ready = False
        if x is not None:
            _lib.call("mp_ep_pack", ptr(x), T, self.d, ptr(self.send_pos), ptr(self.sendbuf), sp)
            self._packed_for = x
            # the receive-side row map needs only the plan: also ahead of the host wait
            _lib.call("mp_ep_recv_layout", self.G, self.T, self.E, self.rank, self.max_slots, None,
                      ptr(self.recv_of_local), ptr(self.ws), self.ws_n, sp)
            self._layout_ready = True
        self.sizes_ready.synchronize()
        host = self.sizes_host.tolist()
        G = self.G
        if host[2 * G] < 0:  # every rank computes the same plan, so every rank raises here
            raise ConfigurationError(f"mp_ep_plan: the layer needs more than max_slots={self.max_slots} slots")
        return EpPlan(host[:G], host[G:2 * G], host[2 * G], self.send_pos[:T], self.piece_row, self.piece_rows,
                      self.exp_begin)

    def pack(self, x: torch.Tensor, plan: EpPlan, n_send: int) -> torch.Tensor:
        if self._packed_for is not x:
            _lib.call("mp_ep_pack", ptr(x), x.shape[0], self.d, ptr(plan.send_pos), ptr(self.sendbuf), stream_ptr())
        self._packed_for = None
        return self.sendbuf[:n_send]

    def recv_buffer(self, n: int) -> torch.Tensor:
        return self.recvbuf[:n]

    def back_buffer(self, n: int) -> torch.Tensor:
        return self.yback[:n]

    def expert_ffn(self, recvbuf: torch.Tensor, plan: EpPlan, l: int, ev=None) -> torch.Tensor:
        n = recvbuf.shape[0]
        # GEMM2 stores (flags bit 5) into the receive-order rows: each row has exactly one writer
        y = self.ybuf[:n]
        if n == 0:
            return y
        lay = self.layers[l]
        if not getattr(self, "_layout_ready", False):
            _lib.call("mp_ep_recv_layout", self.G, self.T, self.E, self.rank, self.max_slots, None,
                      ptr(self.recv_of_local), ptr(self.ws), self.ws_n, stream_ptr())
        self._layout_ready = False
        # xperm region of the FFN workspace <- received rows in local (slot-major) order (fixed
        # splits: the number of local rows stays on the device)
        _lib.call("mp_gather_rows_bf16_dn", ptr(recvbuf), n, self.d, ptr(self.recv_of_local),
                  ptr(self.nloc) if self.peer_cap else None, ptr(self.ffn_ws), stream_ptr())
        sp = stream_ptr()
        if ev is not None:
            ev[0].record(sp)
        # single-CTA grouped GEMMs over the EP pieces (split_m = 1); a V tiled for the CTA-pair
        # kernels (256-column slices) is read with 256-column units (flags bit 6)
        vflag = 64 if lay.tiled and getattr(lay, "vbn", 0) == 256 else 0
        _lib.call("mp_ffn_up", n, self.d, self.F, self.E, ptr(lay.U), lay.tiled, ptr(plan.piece_row),
                  ptr(plan.piece_rows), ptr(plan.exp_begin), ptr(self.ffn_ws), self.ffn_n, sp)
        if ev is not None:
            ev[1].record(sp)
        _lib.call("mp_ffn_down", ptr(y), n, self.d, self.F, self.E, ptr(lay.V), lay.tiled | 32 | vflag,
                  ptr(self.recv_of_local),
                  ptr(plan.piece_row), ptr(plan.piece_rows), ptr(plan.exp_begin), ptr(self.ffn_ws), self.ffn_n, sp)
        if ev is not None:
            ev[2].record(sp)
        return y

    def combine(self, x: torch.Tensor, yback: torch.Tensor, plan: EpPlan) -> None:
        _lib.call("mp_ep_combine", ptr(x), x.shape[0], self.d, ptr(yback), ptr(plan.send_pos), stream_ptr())


class ExpertParallelMoE:
    """The MoE layer stack of one rank; ``forward`` runs all layers on the local token shard."""

    def __init__(self, kernels, num_layers: int, num_experts: int, group=None):
        self.k = kernels
        self.group = group
        self.G = dist.get_world_size(group) if dist.is_initialized() else 1
        self.L, self.E = num_layers, num_experts
        self.force_collectives = False  # tests: NCCL calls even when G == 1
        # residency state (replicated on every rank, updated identically)
        self.res = torch.zeros(num_layers, num_experts, dtype=torch.int32, device=getattr(kernels, "dev", "cpu"))

    def _all_gather_counts(self, counts: torch.Tensor) -> torch.Tensor:
        if self.G == 1 and not self.force_collectives:
            return counts.view(1, -1)
        parts = [torch.empty_like(counts) for _ in range(self.G)]
        dist.all_gather(parts, counts, group=self.group)
        return torch.stack(parts)

    def _a2a(self, out: torch.Tensor, inp: torch.Tensor, out_splits, in_splits) -> None:
        if self.G == 1 and not self.force_collectives:
            out.copy_(inp)
            return
        dist.all_to_all_single(out, inp, output_split_sizes=out_splits, input_split_sizes=in_splits, group=self.group)

    def layer(self, l: int, x: torch.Tensor, ev=None) -> torch.Tensor:
        k = self.k
        route = k.route(x, l)
        if getattr(k, "p2p", False) and k.peer_cap and self.G > 1:
            C = k.allgather_counts_peer(k.counts(route))  # peer stores + device barrier
        else:
            C = self._all_gather_counts(k.counts(route))
        if getattr(k, "p2p", False) and k.peer_cap:
            # peer memory: rows to the destinations, barrier, GEMMs whose epilogue adds the results
            # into the home streams, barrier (the next layer's router reads them)
            plan = k.plan(route, C, self.res[l])
            k.register_stream(x)
            timed = ev is not None and len(ev) >= 7
            if timed:
                ev[3].record(stream_ptr())
            k.dispatch_peer(x, plan)
            k.barrier()
            if timed:
                ev[4].record(stream_ptr())
            k.expert_ffn_peer(plan, l, ev)
            if timed:
                ev[5].record(stream_ptr())
            k.barrier()
            if timed:
                ev[6].record(stream_ptr())
            self.last_route = route
            return x
        early = hasattr(k, "recv_buffer")  # device kernels: pack before the host reads the split sizes
        plan = k.plan(route, C, self.res[l], x) if early else k.plan(route, C, self.res[l])
        sendbuf = k.pack(x, plan, sum(plan.send_counts))
        n_recv = sum(plan.recv_counts)
        recvbuf = k.recv_buffer(n_recv) if early else \
            torch.empty(n_recv, x.shape[1], dtype=sendbuf.dtype, device=sendbuf.device)
        timed = ev is not None and len(ev) >= 7  # events 3..6 bracket the dispatch and combine all-to-alls
        if timed:
            ev[3].record(stream_ptr())
        self._a2a(recvbuf, sendbuf, plan.recv_counts, plan.send_counts)
        if timed:
            ev[4].record(stream_ptr())
        y = k.expert_ffn(recvbuf, plan, l, ev) if ev is not None else k.expert_ffn(recvbuf, plan, l)
        n_send = sum(plan.send_counts)
        yback = k.back_buffer(n_send) if early else torch.empty(n_send, x.shape[1], dtype=y.dtype, device=y.device)
        if timed:
            ev[5].record(stream_ptr())
        self._a2a(yback, y, plan.send_counts, plan.recv_counts)
        if timed:
            ev[6].record(stream_ptr())
        k.combine(x, yback, plan)
        self.last_route = route
        return x

    def forward(self, x: torch.Tensor) -> torch.Tensor:
        for l in range(self.L):
            self.layer(l, x)
        return x
