"""Device plumbing: torch supplies CUDA memory and the current stream.

torch is used only as an allocator / copy engine here; every computation on
matrix data goes through libb2sr_sm100.so.
"""

from __future__ import annotations

import os
import sys
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


class _PinnedBlock:
    __slots__ = ("tensor", "root", "size")

    def __init__(self, size: int):
        t = torch()
        self.tensor = t.empty(size, dtype=t.uint8, pin_memory=True)
        self.root = self.tensor.numpy()  # every array handed out is a view of root
        self.size = size

    def free(self) -> bool:
        # references: this attribute + getrefcount's argument; any live result
        # array (or a view of one) holds one more -- numpy collapses view bases
        return sys.getrefcount(self.root) <= 2


class _PinnedPool:
    """Page-locked result buffers, recycled once the caller drops the array.

    A device->host result copied straight into page-locked memory runs at the
    PCIe rate; copying it into a fresh numpy array afterwards costs several
    times more (first-touch page faults + a host memcpy).  So result arrays
    ARE views of pinned blocks: a block is reused when no array or view of it
    is alive any more.  Bounded (B2SR_PINNED_POOL_MB, default 2048); past the
    bound, results go through one reused staging buffer instead.
    """

    GRAIN = 2 << 20

    def __init__(self):
        self.blocks: list[_PinnedBlock] = []
        self.bytes = 0
        self.cap = int(os.environ.get("B2SR_PINNED_POOL_MB", "2048")) << 20
        self.lock = threading.Lock()

    def lease(self, nbytes: int):
        """(block, view of its first nbytes) of a free block, or None (over the
        bound).  The view is taken under the lock: it is the reference that
        marks the block busy, so no other thread can lease it meanwhile."""
        with self.lock:
            b = self._pick(nbytes)
            return None if b is None else (b, b.root[:nbytes])

    def _pick(self, nbytes: int):
        """Smallest free block that fits (caller holds the lock), else a new one."""
        best = None
        for b in self.blocks:
            if nbytes <= b.size <= 2 * nbytes + self.GRAIN and b.free() and (best is None or b.size < best.size):
                best = b
        if best is not None:
            return best
        size = (nbytes + self.GRAIN - 1) // self.GRAIN * self.GRAIN
        if self.bytes + size > self.cap:
            for b in list(self.blocks):  # make room from free blocks of other sizes
                if self.bytes + size <= self.cap:
                    break
                if b.free():
                    self.blocks.remove(b)
                    self.bytes -= b.size
            if self.bytes + size > self.cap:
                return None
        b = _PinnedBlock(size)
        self.blocks.append(b)
        self.bytes += size
        return b


_pool = _PinnedPool()


def to_host(tensor, dtype, count: int) -> np.ndarray:
    """Copy the first ``count`` elements of ``dtype`` out of a device buffer.

    One DMA into a page-locked block of the result pool; the returned array
    is a view of that block (see _PinnedPool).  Without a block (pool bound
    reached): DMA into a reused staging buffer, then a host copy.
    """
    global _bounce
    t = torch()
    dt = np.dtype(dtype)
    nbytes = count * dt.itemsize
    if nbytes == 0:
        return np.empty(count, dt)
    src = tensor.detach().view(t.uint8)[:nbytes]
    leased = _pool.lease(nbytes)
    if leased is not None:
        blk, view = leased
        blk.tensor[:nbytes].copy_(src)
        return view.view(dt)
    out = np.empty(count, dt)
    with _bounce_lock:
        if _bounce is None or _bounce.numel() < nbytes:
            _bounce = t.empty(max(nbytes, 1 << 20), dtype=t.uint8, pin_memory=True)
        _bounce[:nbytes].copy_(src)
        out.view(np.uint8)[:] = _bounce[:nbytes].numpy()
    return out


_bounce = None  # staging buffer for results past the pool bound
_bounce_lock = threading.Lock()


def ptr(tensor) -> int:
    return tensor.data_ptr()


def padded_vec_bytes(ntr: int, d: int) -> int:
    wb = 4 if d == 32 else (2 if d == 16 else 1)
    return max(4, (ntr * wb + 3) // 4 * 4)
