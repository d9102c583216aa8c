"""bin-SpMV / bin-SpGEMM over B2SR on the B200 (drop-in for b2sr/kernels.py).

Names follow the reference's (matrix, input vector, output vector) precision
triplets.  Every function validates its arguments exactly like the
reference (same exception classes, same order), then runs one sm_100a
kernel through the C ABI:

  =========================  ====================================  ==============
  reference                  kernel (csrc/)                        output
  =========================  ====================================  ==============
  bmv_bin_bin_bin   :97      K4 k_bmv_bbb_stream (bmv_stream.cu)   BitVector
  bmv_bin_bin_full  :118     K5 k_bmv_bbf  (bmv.cu)                float64[n]
  bmv_bin_full_full :140     K6 k_bff_rows + k_vlong_* (bmv_bff.cu, float64[n]
                                bmv_vlong.cu)
  *_masked          :219-249 same kernels, keep fused at store
  bmm_bin_bin_sum   :298     K7 colsum/rowdeg dot (bmm.cu)         int
  bmm_..._masked    :323     K8 k_bmm_masked_items (bmm.cu)        int
  =========================  ====================================  ==============

``workers`` is accepted and validated for signature parity
(resolve_workers); it does not change the computation -- results are
identical for every worker count, as the reference guarantees.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import _device as dev
from .formats import B2srMatrix, BitVector, b2sr_transpose
from .semirings import Semiring

WORKERS_ENV = "BITBLAS_THREADS"


def resolve_workers(workers: int | None = None) -> int:
    """Explicit argument, else $BITBLAS_THREADS, else 1 (kernels.py:33-41)."""
    if workers is None:
        env = os.environ.get(WORKERS_ENV, "").strip()
        workers = int(env) if env else 1
    workers = int(workers)
    if workers < 1:
        raise ValueError("worker count must be at least 1")
    return workers


# ---------------------------------------------------------------- validation
def _bits_operand(a: B2srMatrix, x) -> BitVector:
    if not isinstance(x, BitVector):
        raise TypeError("expected a BitVector input")
    if x.n != a.n or x.dim != a.dim:
        raise ValueError("vector length/tile width must match the matrix")
    return x


def _full_operand(a: B2srMatrix, x) -> np.ndarray:
    if isinstance(x, BitVector):
        raise TypeError("expected a full-precision vector, not a BitVector")
    v = np.asarray(x, dtype=np.float64).reshape(-1) if np.ndim(x) else np.asarray([x], np.float64)
    if v.shape != (a.n,):
        raise ValueError(f"expected a length-{a.n} vector")
    return v


def _keep_operand(a: B2srMatrix, keep) -> BitVector:
    if not isinstance(keep, BitVector):
        raise TypeError("keep mask must be a BitVector")
    if keep.n != a.n or keep.dim != a.dim:
        raise ValueError("keep mask length/tile width must match the matrix")
    return keep


def _words_to_device(v: BitVector):
    return dev.to_device(v.words, pad_bytes=dev.padded_vec_bytes(len(v.words), v.dim))


# ---------------------------------------------------------------- used columns
def used_columns(a: B2srMatrix) -> np.ndarray:
    """Columns holding at least one set bit (kernels.py:86-94)."""
    out = dev.empty_bytes(a.n)
    _capi.call("b2sr_used_columns", a.handle().ptr, dev.ptr(out), dev.stream())
    return dev.to_host(out, np.uint8, a.n).astype(bool)


# ---------------------------------------------------------------- K4
def _bbb(a: B2srMatrix, x: BitVector, keep: BitVector | None) -> BitVector:
    h = a.handle()
    xd = _words_to_device(x)
    kd = _words_to_device(keep) if keep is not None else None
    nbytes = dev.padded_vec_bytes(a.n_tile_rows, a.dim)
    y = dev.empty_bytes(nbytes)
    _capi.call("b2sr_bmv_bbb", h.ptr, dev.ptr(xd), dev.ptr(kd) if kd is not None else None, dev.ptr(y),
               dev.stream())
    words = dev.to_host(y, a.tile_dim.word_dtype, a.n_tile_rows)
    return BitVector(a.n, a.tile_dim, words)


def bmv_bin_bin_bin(a: B2srMatrix, x: BitVector, *, workers: int | None = None) -> BitVector:
    """y[i] = OR_j (a[i,j] AND x[j])."""
    x = _bits_operand(a, x)
    resolve_workers(workers)
    return _bbb(a, x, None)


def bmv_bin_bin_bin_masked(a: B2srMatrix, x: BitVector, keep: BitVector, *,
                           workers: int | None = None) -> BitVector:
    """bmv_bin_bin_bin with cleared keep bits forced to 0 at store time."""
    _keep_operand(a, keep)
    x = _bits_operand(a, x)
    resolve_workers(workers)
    return _bbb(a, x, keep)


# ---------------------------------------------------------------- K5
def _bbf(a: B2srMatrix, x: BitVector, keep: BitVector | None) -> np.ndarray:
    h = a.handle()
    xd = _words_to_device(x)
    kd = _words_to_device(keep) if keep is not None else None
    y = dev.empty_bytes(8 * a.n)
    _capi.call("b2sr_bmv_bbf", h.ptr, dev.ptr(xd), dev.ptr(kd) if kd is not None else None, dev.ptr(y),
               dev.stream())
    return dev.to_host(y, np.float64, a.n)


def bmv_bin_bin_full(a: B2srMatrix, x: BitVector, *, workers: int | None = None) -> np.ndarray:
    """y[i] = number of j with a[i,j] AND x[j], as float64."""
    x = _bits_operand(a, x)
    resolve_workers(workers)
    return _bbf(a, x, None)


def bmv_bin_bin_full_masked(a: B2srMatrix, x: BitVector, keep: BitVector, *,
                            workers: int | None = None) -> np.ndarray:
    """bmv_bin_bin_full with cleared keep positions forced to 0."""
    _keep_operand(a, keep)
    x = _bits_operand(a, x)
    resolve_workers(workers)
    return _bbf(a, x, keep)


# ---------------------------------------------------------------- K6
def _bff(a: B2srMatrix, x, semiring: Semiring, scale, keep: BitVector | None) -> np.ndarray:
    xv = _full_operand(a, x)
    if semiring.name == "boolean":
        raise ValueError("boolean semiring has no full-precision gather; use bmv_bin_bin_bin")
    sc = None
    if scale is not None:
        if semiring.name != "arithmetic":
            raise ValueError("scale is only supported with the arithmetic semiring")
        sc = np.asarray(scale, dtype=np.float64).reshape(-1)
        if sc.shape != (a.n,):
            raise ValueError(f"expected a length-{a.n} scale vector")
    h = a.handle()
    xd = dev.to_device(xv)
    sd = dev.to_device(sc) if sc is not None else None
    kd = _words_to_device(keep) if keep is not None else None
    y = dev.empty_bytes(8 * a.n)
    bad = ctypes.c_int64(-1)
    # the semiring's own add identity (kernels.py:176, 249): any float the
    # public Semiring constructor accepts, e.g. Semiring("maxtimes", -inf)
    _capi.call("b2sr_bmv_bff_ex", h.ptr, dev.ptr(xd), _capi.RING[semiring.name], float(semiring.edge_increment),
               float(semiring.add_identity), dev.ptr(sd) if sd is not None else None,
               dev.ptr(kd) if kd is not None else None, dev.ptr(y), ctypes.addressof(bad), dev.stream())
    return dev.to_host(y, np.float64, a.n)


def bmv_bin_full_full(a: B2srMatrix, x, semiring: Semiring, scale=None, *,
                      workers: int | None = None) -> np.ndarray:
    """Semiring gather y[i] = reduce over set a[i,j] of x[j] (ascending j)."""
    if isinstance(x, BitVector):
        raise TypeError("expected a full-precision vector, not a BitVector")
    _full_operand(a, x)
    if semiring.name == "boolean":
        raise ValueError("boolean semiring has no full-precision gather; use bmv_bin_bin_bin")
    resolve_workers(workers)
    return _bff(a, x, semiring, scale, None)


def bmv_bin_full_full_masked(a: B2srMatrix, x, semiring: Semiring, keep: BitVector, scale=None, *,
                             workers: int | None = None) -> np.ndarray:
    """bmv_bin_full_full with cleared keep positions holding the add identity."""
    _keep_operand(a, keep)
    _full_operand(a, x)
    if semiring.name == "boolean":
        raise ValueError("boolean semiring has no full-precision gather; use bmv_bin_bin_bin")
    resolve_workers(workers)
    return _bff(a, x, semiring, scale, keep)


@dataclass(frozen=True)
class MaskedOutput:
    """A masked result bundled with its keep mask, for auditing (kernels.py:252-268)."""

    result: object
    keep: BitVector

    def cleared_values(self) -> np.ndarray:
        off = ~self.keep.to_bools()
        if isinstance(self.result, BitVector):
            return self.result.to_bools()[off].astype(np.float64)
        return np.asarray(self.result)[off]


# ---------------------------------------------------------------- K7 / K8
def _check_bmm(a: B2srMatrix, b):
    if not isinstance(b, B2srMatrix):
        raise TypeError("expected a B2srMatrix operand")
    if a.n != b.n or a.dim != b.dim:
        raise ValueError("operands must share n and tile width")
    if a.n ** 3 > 2 ** 63 - 1:
        raise ValueError("entry-sum may overflow a 64-bit accumulator")


def bmm_bin_bin_sum(a: B2srMatrix, b: B2srMatrix, *, workers: int | None = None) -> int:
    """Sum of all entries of the integer product A @ B."""
    _check_bmm(a, b)
    resolve_workers(workers)
    out = ctypes.c_int64()
    _capi.call("b2sr_bmm_sum", a.handle().ptr, b.handle().ptr, ctypes.addressof(out), dev.stream())
    return int(out.value)


def bmm_bin_bin_sum_masked(a: B2srMatrix, b: B2srMatrix, mask: B2srMatrix, *,
                           workers: int | None = None) -> int:
    """Sum of (A @ B)[i, j] over the positions where mask[i, j] = 1."""
    _check_bmm(a, b)
    _check_bmm(a, mask)
    resolve_workers(workers)
    if mask.num_tiles == 0:
        return 0
    bt = b2sr_transpose(b)
    out = ctypes.c_int64()
    _capi.call("b2sr_bmm_sum_masked_bt", a.handle().ptr, bt.handle().ptr, mask.handle().ptr,
               ctypes.addressof(out), dev.stream())
    return int(out.value)
