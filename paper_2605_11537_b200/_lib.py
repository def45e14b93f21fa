"""ctypes binding of ``libmoempmc.so`` (include/moempmc.h).

This is the only way the Python layer reaches the GPU kernels. There is no
CPU fallback: if the library or a CUDA device is missing, every entry point
raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import (
    ConfigurationError,
    DeviceError,
    InfeasibleCapacityError,
    NumericError,
    PlacementError,
)

LIB_PATH = Path(__file__).resolve().with_name("libmoempmc.so")

MP_OK, MP_ERR_CONFIG, MP_ERR_NUMERIC, MP_ERR_PLACEMENT, MP_ERR_INFEASIBLE, MP_ERR_CUDA = range(6)
MP_EVENT_NONE = -1
MP_EVENT_KIND_SHIFT = 24
MP_EVENT_LOAD = 1
MP_EVENT_REPLICATE = 2

_P = ctypes.c_void_p
_I = ctypes.c_int
_Z = ctypes.c_size_t
_F = ctypes.c_float
_D = ctypes.c_double

# name -> (restype, argtypes); mirrors include/moempmc.h
SIGNATURES: dict[str, tuple] = {
    "mp_abi_version": (_I, []),
    "mp_last_error": (ctypes.c_char_p, []),
    "mp_device_info": (_I, [_P, _P, _P]),
    "mp_histogram": (_I, [_P, _I, _I, _I, _P, _P]),
    "mp_histogram_workspace_bytes": (_Z, [_I, _I, _I]),
    "mp_histogram_ws": (_I, [_P, _I, _I, _I, _P, _P, _Z, _P]),
    "mp_cap_replicas": (_I, [_P, _I, _I, _I, _I, _P, _P, _P]),
    "mp_place_workspace_bytes": (_Z, [_I, _I, _I]),
    "mp_place": (_I, [_P, _I, _I, _I, _P, _I, _I, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_exec_workspace_bytes": (_Z, [_I, _I, _I, _I]),
    "mp_set_sm_partition": (_I, [_I, _I]),
    "mp_exec_map": (_I, [_P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_exec_map_hist": (_I, [_P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _I, _P, _P, _Z, _P]),
    "mp_gemm_bf16": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _I, _P]),
    "mp_sru_workspace_bytes": (_Z, [_I, _I]),
    "mp_sru_layer": (_I, [_P, _P, _P, _P, _I, _I, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_sru_project": (_I, [_P, _P, _P, _I, _I, _P, _Z, _P]),
    "mp_sru_scan": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_sru_train_fwd": (_I, [_P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P]),
    "mp_sru_train_bwd": (_I, [_P, _P, _P, _P, _P, _P, _P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P]),
    "mp_train_colsum": (_I, [_P, _I, _I, _P, _P]),
    "mp_train_ce": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "mp_train_sum": (_I, [_P, _I, _P, _P]),
    "mp_train_axpy": (_I, [_P, _P, _Z, _D, _P]),
    "mp_dgemm": (_I, [_I, _I, _I, _I, _I, _P, _I, _P, _I, _D, _P, _I, _P]),
    "mp_train_nonfinite": (_I, [_P, _Z, _P, _P]),
    "mp_sru_scan_total": (_I, [_I, _I, _P, _P, _Z, _P]),
    "mp_sru_fold_carry": (_I, [_P, _I, _I, _P, _P, _P]),
    "mp_sru_scan_finish": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_sparsemax_rows": (_I, [_P, _I, _I, _P, _P]),
    "mp_segments_workspace_bytes": (_Z, [_I, _I]),
    "mp_segments_from_slots": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_heads_argmax": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _P]),
    "mp_router_workspace_bytes": (_Z, [_I, _I]),
    "mp_route_top1": (_I, [_P, _I, _I, _I, _P, _P, _I, _I, _F, _P, _P, _Z, _P]),
    "mp_router_weight_absmax": (_I, [_P, _I, _I, _P, _P]),
    "mp_route_top1_ex": (_I, [_P, _I, _I, _I, _P, _P, _P, _I, _I, _P, _P, _Z, _P]),
    "mp_route_top1_hist": (_I, [_P, _I, _I, _I, _P, _P, _P, _I, _I, _P, _P, _P, _Z, _P]),
    "mp_ffn_workspace_bytes": (_Z, [_I, _I, _I]),
    "mp_moe_ffn": (_I, [_P, _P, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_ffn_gather": (_I, [_P, _I, _I, _I, _I, _P, _P, _Z, _P]),
    "mp_ffn_up": (_I, [_I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _Z, _P]),
    "mp_ffn_down": (_I, [_P, _I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_ffn_down_bn": (_I, [_I]),
    "mp_ffn_up_bn": (_I, [_I]),
    "mp_pool_state_bytes": (_Z, [_I, _I, _I]),
    "mp_pool_init": (_I, [_I, _I, _I, _P, _P]),
    "mp_pool_update": (_I, [_P, _I, _I, _I, _P, _P]),
    "mp_replica_copy": (_I, [_P, _P, _P, _P, _Z, _I, _P, _I, _I, _P]),
    "mp_piece_pool": (_I, [_P, _P, _I, _P, _P, _P, _I, _I, _P, _I, _P]),
    "mp_pool_stats": (_I, [_P, _I, _I, _I, _P, _P]),
    "mp_ffn_up_pool": (_I, [_I, _I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_ffn_down_pool": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_debug_cta_times": (_I, [_P, _P, _I]),
    "mp_layer_counts": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P]),
    "mp_tile_kmajor": (_I, [_P, _P, _I, _I, _I, _I, _P]),
    "mp_ep_workspace_bytes": (_Z, [_I, _I, _I, _I]),
    "mp_ep_plan": (_I, [_P, _I, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_ep_pack": (_I, [_P, _I, _I, _P, _P, _P]),
    "mp_ep_recv_layout": (_I, [_I, _I, _I, _I, _I, _P, _P, _P, _Z, _P]),
    "mp_gather_rows_bf16": (_I, [_P, _I, _I, _P, _P, _P]),
    "mp_ep_combine": (_I, [_P, _I, _I, _P, _P, _P]),
    "mp_ep_plan_cap": (_I, [_P, _I, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_gather_rows_bf16_dn": (_I, [_P, _I, _I, _P, _P, _P, _P]),
    "mp_ep_pack_peer": (_I, [_P, _I, _I, _P, _I, _I, _P, _P, _P]),
    "mp_peer_barrier": (_I, [_P, _I, _I, _P, _P, _P]),
    "mp_peer_allgather_i32": (_I, [_P, _I, _I, _I, _I, _P, _I, _P]),
    "mp_ep_gather_peer": (_I, [_P, _I, _I, _P, _P, _P, _I, _I, _P, _P, _P]),
    "mp_ffn_down_peer": (_I, [_P, _I, _I, _I, _I, _I, _P, _I, _P, _P, _P, _P, _P, _Z, _P]),
    "mp_f32_to_bf16": (_I, [_P, _P, _Z, _P]),
    "mp_l2_persist": (_I, [_P, _Z, _F, _P]),
    "mp_enable_peer_access": (_I, [_I]),
    "mp_graph_begin": (_I, [_P]),
    "mp_graph_end": (_I, [_P, _P]),
    "mp_graph_end_counted": (_I, [_P, _P, _P]),
    "mp_graph_launch": (_I, [_P, _P]),
    "mp_graph_destroy": (_I, [_P]),
    "mp_event_create": (_I, [_P]),
    "mp_event_record": (_I, [_P, _P]),
    "mp_event_elapsed_ms": (_I, [_P, _P, _P]),
    "mp_event_destroy": (_I, [_P]),
}

_ERRORS = {
    MP_ERR_CONFIG: ConfigurationError,
    MP_ERR_NUMERIC: NumericError,
    MP_ERR_PLACEMENT: PlacementError,
    MP_ERR_INFEASIBLE: InfeasibleCapacityError,
    MP_ERR_CUDA: DeviceError,
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load_library(path: Path | str | None = None) -> ctypes.CDLL:
    """Load (once) and type the native library. Does not touch the GPU."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path is not None else LIB_PATH
        if not p.exists():
            raise DeviceError(
                f"native library {p} is missing; build it with "
                "`python -m paper_2605_11537_b200.build` (nvcc, sm_100a)"
            )
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    return list(SIGNATURES)


def check(status: int, what: str = "") -> None:
    """Map a C-ABI status onto the reference exception classes."""
    if status == MP_OK:
        return
    msg = (load_library().mp_last_error() or b"").decode(errors="replace")
    exc = _ERRORS.get(status, DeviceError)
    raise exc(f"{what}: {msg}" if what else msg)


def call(name: str, *args) -> int:
    """Call an int-returning entry point and raise on a non-OK status."""
    fn = getattr(load_library(), name)
    status = fn(*args)
    check(status, name)
    return status


def size_query(name: str, *args) -> int:
    return int(getattr(load_library(), name)(*args))
