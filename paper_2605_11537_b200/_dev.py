"""Device plumbing shared by the host API: CUDA checks, streams, workspaces.

PyTorch is used only for device memory, streams and events; every computation
on the hot path is a call into ``libmoempmc.so``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .errors import DeviceError

_checked = False


def require_device() -> torch.device:
    """The CUDA device the kernels run on; raises if there is none (no CPU fallback)."""
    global _checked
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the MoE-MPMC hot path runs only on sm_100a (B200)")
    if not _checked:
        _lib.load_library()
        major, minor = torch.cuda.get_device_capability()
        if (major, minor) != (10, 0):
            raise DeviceError(f"libmoempmc.so is built for sm_100a; device is sm_{major}{minor}")
        _checked = True
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr(stream: torch.cuda.Stream | None = None) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise DeviceError("expected a CUDA tensor")
    return int(t.data_ptr())


def to_device_i32(a, dev) -> torch.Tensor:
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=torch.int32).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(dev)


class Workspace:
    """Grow-only device scratch buffers keyed by purpose."""

    def __init__(self) -> None:
        self._bufs: dict[str, torch.Tensor] = {}

    def get(self, key: str, nbytes: int, device: torch.device) -> torch.Tensor:
        nbytes = max(int(nbytes), 256)
        buf = self._bufs.get(key)
        if buf is None or buf.numel() < nbytes or buf.device != device:
            buf = torch.empty(nbytes, dtype=torch.uint8, device=device)
            self._bufs[key] = buf
        return buf


WORKSPACE = Workspace()


class _Staging:
    """Two page-locked bounce buffers for host -> device copies of pageable (numpy) arrays:
    the host copy of chunk i overlaps the DMA of chunk i - 1 (50 MB: ~1.6 ms against ~2.6-3.6 ms
    for a pageable copy and ~6.7 ms for registering the array's pages)."""

    CHUNK = 4 << 20

    def __init__(self):
        self.pin = None
        self.ev = None

    def to_device(self, src: torch.Tensor, dev) -> torch.Tensor:
        out = torch.empty(src.shape, dtype=src.dtype, device=dev)
        n = src.numel() * src.element_size()
        if n < 2 * self.CHUNK:
            out.copy_(src)
            return out
        if self.pin is None:
            self.pin = [torch.empty(self.CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(2)]
            self.ev = [torch.cuda.Event(), torch.cuda.Event()]
        s8, d8 = src.view(-1).view(torch.uint8), out.view(-1).view(torch.uint8)
        for k, i in enumerate(range(0, n, self.CHUNK)):
            j, m = k % 2, min(self.CHUNK, n - i)
            self.ev[j].synchronize()  # the DMA that last read this buffer is done
            self.pin[j][:m].copy_(s8[i:i + m])
            d8[i:i + m].copy_(self.pin[j][:m], non_blocking=True)
            self.ev[j].record()
        return out


_STAGING_TLS = __import__("threading").local()  # one pair of bounce buffers per host thread


def _staging() -> _Staging:
    st = getattr(_STAGING_TLS, "st", None)
    if st is None:
        st = _STAGING_TLS.st = _Staging()
    return st


def upload_rows(arr, d: int, dp: int, dev, name: str = "embeddings") -> torch.Tensor:
    """(T, d) float rows -> (T, dp) float32 device tensor, zero padded. Non-finite values raise
    NumericError like src/validation.py:22-27, checked on the device (one flag read) instead of
    a host pass over the array; float64 input is narrowed on the device."""
    from .errors import NumericError

    a = np.asarray(arr)
    if a.dtype not in (np.float32, np.float64):
        a = a.astype(np.float32)
    a = np.ascontiguousarray(a)
    t = _staging().to_device(torch.from_numpy(a), dev)
    if not bool(torch.isfinite(t).all().item()):
        raise NumericError(f"{name} contains non-finite values")
    if t.ndim != 2 or t.shape[1] != d:
        return t  # the caller reports the shape error
    if dp == d and t.dtype == torch.float32:
        return t
    out = torch.zeros(t.shape[0], dp, dtype=torch.float32, device=dev)
    out[:, :d] = t
    return out


def download(t: torch.Tensor) -> np.ndarray:
    """Device tensor -> numpy through page-locked memory (torch's caching host allocator reuses
    the pinned block once the array is released): a pageable D2H of a 50 MB stream runs at
    ~2 GB/s, a pinned one at PCIe speed."""
    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t)
    return out.numpy()


def round_up(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def pow2_at_least(x: int, lo: int) -> int:
    p = lo
    while p < x:
        p *= 2
    return p
