"""CPU-only checks of the drop-in boundary: the sm_100a library loads (no GPU
needed to dlopen it), exports every symbol include/moempmc.h declares, and the
ctypes signature table matches the header. Also: the product package refuses to
run without a CUDA device instead of falling back to the CPU."""

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "moempmc.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"MP_API\s+(?:const\s+)?\w+\**\s+\**(mp_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_11537_b200.build import build

    build()
    from paper_2605_11537_b200 import _lib

    return _lib.load_library()


def test_header_declares_the_hot_path(lib):
    syms = declared_symbols()
    for must in ("mp_histogram", "mp_cap_replicas", "mp_place", "mp_exec_map", "mp_sru_layer", "mp_heads_argmax",
                 "mp_route_top1", "mp_moe_ffn", "mp_replica_copy", "mp_gemm_bf16"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    from paper_2605_11537_b200 import _lib

    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (mp_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    for s in declared_symbols():
        assert isinstance(getattr(lib, s), ctypes._CFuncPtr)


def test_ctypes_table_matches_header(lib):
    from paper_2605_11537_b200 import _lib

    text = HEADER.read_text()
    for name, (_, args) in _lib.SIGNATURES.items():
        m = re.search(r"MP_API\s+[\w\s\*]+?\b" + name + r"\s*\(([^)]*)\)", text)
        assert m, f"{name} not declared in the header"
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), (name, len(params), len(args))
    assert set(_lib.SIGNATURES) == set(declared_symbols())


def test_abi_version_and_error_string(lib):
    assert lib.mp_abi_version() == 1
    assert isinstance(lib.mp_last_error(), bytes)


def test_size_queries_are_pure_host(lib):
    # workspace sizing never touches the device
    assert lib.mp_place_workspace_bytes(12, 16384, 128) >= 12 * 128 * 128 * 4
    assert lib.mp_exec_workspace_bytes(1, 16384, 128, 424) > 0
    assert lib.mp_ffn_workspace_bytes(16384, 768, 3072) >= 16384 * 768 * 2 + 16384 * 3072 * 2
    assert lib.mp_sru_workspace_bytes(16384, 768) >= 16384 * 3 * 768 * 2
    assert lib.mp_ffn_down_bn(768) == 192 and lib.mp_ffn_down_bn(512) == 256
    assert lib.mp_ffn_down_bn(128) == 128 and lib.mp_ffn_down_bn(64) == 64
    assert lib.mp_ffn_up_bn(3072) == 256


def test_config_errors_map_to_reference_exceptions(lib):
    from paper_2605_11537_b200 import ConfigurationError, _lib

    # argument validation happens before any device work
    with pytest.raises(ConfigurationError):
        _lib.call("mp_cap_replicas", None, 1, 4, 0, 1, None, None, None)
    with pytest.raises(ConfigurationError):
        _lib.call("mp_gemm_bf16", None, None, None, 10, 100, 64, 0, 100, None, 0, 0, None)
    with pytest.raises(ConfigurationError):
        _lib.call("mp_sru_layer", None, None, None, None, 0, 64, None, None, None, None, None, None, 0, None)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2605_11537_b200 import DeviceError
    from paper_2605_11537_b200.planner import cap_replicas
    from paper_2605_11537_b200.predictor import HashTable

    with pytest.raises(DeviceError):
        cap_replicas({0: 5, 1: 3}, 4)
    with pytest.raises(DeviceError):
        HashTable.from_assignment(0, np.array([[0, 1, 1]]))
