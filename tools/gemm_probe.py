"""GEMM micro-probe: libmoempmc dense tcgen05 GEMM vs cuBLAS on the hot-path shapes."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2605_11537_b200 import _lib  # noqa: E402
from paper_2605_11537_b200._dev import ptr, require_device, stream_ptr  # noqa: E402


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3  # us


def main():
    dev = require_device()
    for (M, N, K) in [(16384, 2304, 768), (16384, 3072, 768), (16384, 768, 3072), (16384, 1536, 768)]:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        bias = torch.randn(N, device=dev)
        fl = 2 * M * N * K
        res = {}
        res["ours_plain"] = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, N, None, 0, 0,
                                                     stream_ptr()))
        res["ours_bias_sig"] = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, N, ptr(bias),
                                                        2, K, stream_ptr()))
        res["ours_nostore"] = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, 0, None, 0, 0,
                                                       stream_ptr()))
        res["cublas"] = timeit(lambda: torch.matmul(A, B.T, out=C))
        print(f"M={M} N={N} K={K}: " + "  ".join(f"{k}={v:.1f}us ({fl / v / 1e6:.0f} TF)" for k, v in res.items()))


if __name__ == "__main__" and not ({"--stream", "--pair", "--epi", "--mma"} & set(sys.argv)):
    main()


def stream_probe():
    """Pure weight streaming: one 128-row M tile against every expert's weights (B >> L2)."""
    dev = require_device()
    for (N, K) in [(128 * 3072, 768), (128 * 768, 3072)]:
        A = torch.randn(128, K, device=dev).bfloat16()
        B = (torch.randn(N, K, device=dev) / 8).bfloat16()
        C = torch.empty(128, N, device=dev, dtype=torch.bfloat16)
        us = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), 128, N, K, 0, N, None, 0, 0,
                                      stream_ptr()), iters=10)
        us0 = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), 128, N, K, 0, 0, None, 0, 0,
                                       stream_ptr()), iters=10)
        X = torch.empty_like(B)
        usc = timeit(lambda: X.copy_(B), iters=10)
        print(f"stream N={N} K={K}: gemm {us:.1f}us = {B.numel() * 2 / us / 1e3:.0f} GB/s of B; nostore {us0:.1f}us "
              f"= {B.numel() * 2 / us0 / 1e3:.0f} GB/s; torch copy {usc:.1f}us = {2 * B.numel() * 2 / usc / 1e3:.0f} GB/s r+w")


if __name__ == "__main__" and "--stream" in sys.argv:
    stream_probe()


def pair_probe():
    """Single-CTA (M = 128) vs CTA-pair (cta_group::2, M = 256) dense GEMM, with and without
    the bf16 store, on the diagnostic build (-DMP_DIAG exports mp_debug_gemm_pair)."""
    import ctypes

    from paper_2605_11537_b200.build import PKG, build

    lib = _lib.load_library(build(extra=["-DMP_DIAG"], out=PKG / "libmoempmc_trace.so"))
    lib.mp_debug_gemm_pair.restype = ctypes.c_int
    lib.mp_debug_gemm_pair.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int] * 4 + [ctypes.c_void_p]
    dev = require_device()
    for (M, N, K) in [(16384, 3072, 768), (16384, 2304, 768), (16384, 768, 3072), (32768, 4096, 4096)]:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        C2 = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        fl = 2 * M * N * K
        res = {}
        res["single"] = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, N, None, 0, 0,
                                                 stream_ptr()))
        res["single_nostore"] = timeit(lambda: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, 0, None,
                                                         0, 0, stream_ptr()))
        res["pair"] = timeit(lambda: _lib.check(lib.mp_debug_gemm_pair(ptr(A), ptr(B), ptr(C2), M, N, K, N,
                                                                       stream_ptr())))
        res["pair_nostore"] = timeit(lambda: _lib.check(lib.mp_debug_gemm_pair(ptr(A), ptr(B), ptr(C2), M, N, K, 0,
                                                                               stream_ptr())))
        res["cublas"] = timeit(lambda: torch.matmul(A, B.T))
        _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, N, None, 0, 0, stream_ptr())
        _lib.check(lib.mp_debug_gemm_pair(ptr(A), ptr(B), ptr(C2), M, N, K, N, stream_ptr()))
        torch.cuda.synchronize()
        same = bool(torch.equal(C, C2))
        print(f"M={M} N={N} K={K}: " + "  ".join(f"{k}={v:.1f}us ({fl / v / 1e6:.0f} TF)" for k, v in res.items())
              + f"  pair==single {same}")


if __name__ == "__main__" and "--pair" in sys.argv:
    pair_probe()


def epi_probe():
    """Where the bf16-store epilogue's cost goes (diagnostic build): TMA bulk stores (product),
    the same epilogue with the store instructions skipped, st.global stores through the smem
    transpose (MP_DIAG_LSU), and no epilogue output at all."""
    import ctypes
    import os

    from paper_2605_11537_b200.build import PKG, build

    lib = _lib.load_library(build(extra=["-DMP_DIAG"], out=PKG / "libmoempmc_trace.so"))
    lib.mp_debug_set_epi.restype = ctypes.c_int
    lib.mp_debug_set_epi.argtypes = [ctypes.c_int]
    dev = require_device()
    for (M, N, K) in [(16384, 3072, 768), (16384, 2304, 768)]:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        fl = 2 * M * N * K
        g = lambda ldc: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(C), M, N, K, 0, ldc, None, 0, 0, stream_ptr())
        res = {"tma": timeit(lambda: g(N))}
        lib.mp_debug_set_epi(1)
        res["tma_pack_only"] = timeit(lambda: g(N))
        lib.mp_debug_set_epi(0)
        os.environ["MP_DIAG_LSU"] = "1"
        res["lsu"] = timeit(lambda: g(N))
        del os.environ["MP_DIAG_LSU"]
        for h in (1, 2):
            os.environ["MP_DIAG_HINT"] = str(h)
            res[f"tma_hint{h}"] = timeit(lambda: g(N))
        del os.environ["MP_DIAG_HINT"]
        res["no_output"] = timeit(lambda: g(0))
        print(f"M={M} N={N} K={K}: " + "  ".join(f"{k}={v:.1f}us ({fl / v / 1e6:.0f} TF)" for k, v in res.items()))


if __name__ == "__main__" and "--epi" in sys.argv:
    epi_probe()


def mma_probe():
    """Shared-memory traffic test (diagnostic build): the dense GEMM with every N = 256 MMA
    issued as two N = 128 MMAs, so the A tile is read from shared memory twice per k-block
    (96 -> 112 KB of shared-memory traffic per k-block, the same MMA work and result). A kernel
    bound by shared-memory bandwidth slows by ~17 %; one bound by the MMA or by TMA does not."""
    import ctypes

    from paper_2605_11537_b200.build import PKG, build

    lib = _lib.load_library(build(extra=["-DMP_DIAG"], out=PKG / "libmoempmc_trace.so"))
    lib.mp_debug_set_mma.restype = ctypes.c_int
    lib.mp_debug_set_mma.argtypes = [ctypes.c_int]
    dev = require_device()
    for (M, N, K) in [(16384, 3072, 768), (16384, 2304, 768), (32768, 4096, 4096)]:
        A = torch.randn(M, K, device=dev).bfloat16()
        B = torch.randn(N, K, device=dev).bfloat16()
        C = torch.empty(M, N, device=dev, dtype=torch.bfloat16)
        C2 = torch.empty_like(C)
        fl = 2 * M * N * K
        g = lambda ldc, out: _lib.call("mp_gemm_bf16", ptr(A), ptr(B), ptr(out), M, N, K, 0, ldc, None, 0, 0,
                                       stream_ptr())
        res = {}
        for flag in (0, 1, 0, 1):
            lib.mp_debug_set_mma(flag)
            res[f"nostore_split{flag}"] = timeit(lambda: g(0, C))
            res[f"store_split{flag}"] = timeit(lambda: g(N, C if flag == 0 else C2))
        lib.mp_debug_set_mma(0)
        torch.cuda.synchronize()
        same = bool(torch.equal(C, C2))
        print(f"M={M} N={N} K={K}: " + "  ".join(f"{k}={v:.1f}us ({fl / v / 1e6:.0f} TF)" for k, v in res.items())
              + f"  split==plain {same}")


if __name__ == "__main__" and "--mma" in sys.argv:
    mma_probe()
