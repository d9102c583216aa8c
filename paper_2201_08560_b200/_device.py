"""Device plumbing: torch supplies CUDA memory and the current stream.

torch is used only as an allocator / copy engine here; every computation on
matrix data goes through libb2sr_sm100.so.
"""

from __future__ import annotations

import threading
import warnings

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def require_cuda():
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError(
            "paper_2201_08560_b200 runs its hot path on a CUDA device (B200, sm_100a); "
            "no GPU is visible and there is no CPU fallback")
    return t


def device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())


def stream() -> int:
    t = require_cuda()
    return t.cuda.current_stream().cuda_stream


def is_cuda_tensor(x) -> bool:
    t = torch()
    return isinstance(x, t.Tensor) and x.is_cuda


def to_device(a: np.ndarray, pad_bytes: int = 0):
    """Upload a host array as raw bytes (padded to 16 B) to the current device.

    Buffers are untyped uint8 tensors; the C ABI receives their pointers and
    the dtype lives on the Python side.
    """
    t = require_cuda()
    a = np.ascontiguousarray(a)
    size = max(a.nbytes, pad_bytes)
    size = (size + 15) // 16 * 16 or 16
    out = t.empty(size, dtype=t.uint8, device=device())
    if a.nbytes:
        with warnings.catch_warnings():  # read-only host arrays are fine to copy from
            warnings.simplefilter("ignore", UserWarning)
            src = t.from_numpy(a.reshape(-1).view(np.uint8))
        out[: a.nbytes].copy_(src, non_blocking=False)
    if size > a.nbytes:
        out[a.nbytes:].zero_()
    return out


def empty_bytes(nbytes: int):
    t = require_cuda()
    return t.empty((int(nbytes) + 15) // 16 * 16 or 16, dtype=t.uint8, device=device())


def zeros_bytes(nbytes: int):
    t = require_cuda()
    return t.zeros((int(nbytes) + 15) // 16 * 16 or 16, dtype=t.uint8, device=device())


def to_host(tensor, dtype, count: int) -> np.ndarray:
    """Copy the first ``count`` elements of ``dtype`` out of a device buffer.

    One DMA into a reused page-locked bounce buffer, then a host copy into the
    fresh result array (measured: a fresh pinned allocation per call costs
    twice as much; the host copy is dominated by first-touch page faults of
    the result, which any new array pays).
    """
    global _bounce
    t = torch()
    dt = np.dtype(dtype)
    nbytes = count * dt.itemsize
    out = np.empty(count, dt)
    if nbytes == 0:
        return out
    with _bounce_lock:
        if _bounce is None or _bounce.numel() < nbytes:
            _bounce = t.empty(max(nbytes, 1 << 20), dtype=t.uint8, pin_memory=True)
        _bounce[:nbytes].copy_(tensor.detach().view(t.uint8)[:nbytes])
        out.view(np.uint8)[:] = _bounce[:nbytes].numpy()
    return out


_bounce = None  # reusable page-locked staging buffer for device -> host copies
_bounce_lock = threading.Lock()


def ptr(tensor) -> int:
    return tensor.data_ptr()


def padded_vec_bytes(ntr: int, d: int) -> int:
    wb = 4 if d == 32 else (2 if d == 16 else 1)
    return max(4, (ntr * wb + 3) // 4 * 4)
