"""B2SR bit-tile storage: host containers with device mirrors.

Drop-in for b2sr/formats.py (reference formats.py:1-554).  The layout is the
reference's, byte for byte: square tiles of width 4/8/16/32 stored as ``dim``
little-endian row words (LSB = lowest column; 1/1/2/4 bytes per word; the
high nibble of 4-wide rows is clear; padding beyond ``n`` is zero).

What changed is where the work happens:
  * ``csr_to_b2sr``, ``b2sr_transpose``, ``b2sr_to_csr`` and the diagonal
    drop run as sm_100a kernels (libb2sr_sm100.so) on device-resident data;
  * a ``B2srMatrix`` built on the device keeps only a device handle; its
    host arrays (``tile_row_ptr`` / ``tile_col_ind`` / ``bit_tiles``) are
    copied down lazily the first time a caller touches them;
  * a ``B2srMatrix`` built from host arrays is validated on the host exactly
    like the reference (FormatError cases of formats.py:242-295) and
    uploaded on first kernel use.
The host-side container code (validation, BitVector, byte accounting, the
``.b2sr`` file format) is plain numpy: it is the boundary, not the hot path.
"""

from __future__ import annotations

import ctypes
import struct
import threading
import weakref
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import _device as dev
from .errors import FormatError

TILE_DIMS = (4, 8, 16, 32)
_WORD = {4: np.dtype("<u1"), 8: np.dtype("<u1"), 16: np.dtype("<u2"), 32: np.dtype("<u4")}
_MAGIC = b"B2SR"
_VERSION = 1
_HEADER = struct.Struct("<4sIIIIQ")  # magic, version, n, dim, n_tile_rows, num_tiles


@dataclass(frozen=True)
class TileDim:
    """A supported tile width (reference formats.py:35-66)."""

    dim: int

    def __post_init__(self):
        if self.dim not in TILE_DIMS:
            raise ValueError(f"tile dim must be one of {TILE_DIMS}, got {self.dim!r}")

    @staticmethod
    def of(dim) -> "TileDim":
        return dim if isinstance(dim, TileDim) else TileDim(int(dim))

    @property
    def word_dtype(self) -> np.dtype:
        return _WORD[self.dim]

    @property
    def row_word_bytes(self) -> int:
        return _WORD[self.dim].itemsize

    @property
    def tile_bytes(self) -> int:
        return self.dim * self.row_word_bytes

    def tile_rows(self, n: int) -> int:
        return -(-int(n) // self.dim)


# ---------------------------------------------------------------- helpers
def _index_array(a, what: str) -> np.ndarray:
    arr = np.asarray(a)
    if arr.ndim != 1:
        raise FormatError(f"{what} must be one-dimensional")
    if arr.size:
        if arr.dtype.kind not in "ui":
            raise FormatError(f"{what} must hold integers")
        lo, hi = int(arr.min()), int(arr.max())
        if lo < 0 or hi > 0xFFFFFFFF:
            raise FormatError(f"{what} entries out of uint32 range")
    out = np.array(arr, dtype=np.uint32, copy=True)
    out.flags.writeable = False
    return out


def _check_ptr(ptr: np.ndarray, length: int, total: int, what: str, length_msg: str, last_msg: str):
    """The row-pointer checks of formats.py:119-127 / 257-263, same messages."""
    if ptr.shape != (length,):
        raise FormatError(length_msg)
    if ptr[0] != 0:
        raise FormatError(f"{what} must start at 0")
    if length > 1 and np.any(ptr[1:] < ptr[:-1]):
        raise FormatError(f"{what} must be non-decreasing")
    if int(ptr[-1]) != total:
        raise FormatError(last_msg)


def _strictly_increasing_in_segments(ptr: np.ndarray, idx: np.ndarray) -> bool:
    """True when idx rises strictly inside every [ptr[i], ptr[i+1]) segment."""
    if len(idx) < 2:
        return True
    step_ok = idx[1:].astype(np.int64) > idx[:-1].astype(np.int64)
    starts = ptr[1:-1].astype(np.int64)
    starts = starts[(starts > 0) & (starts < len(idx))]
    step_ok[starts - 1] = True  # a new segment may restart low
    return bool(step_ok.all())


def _pack_rows(bits01: np.ndarray, d: int) -> np.ndarray:
    """(..., d) 0/1 -> row words (bit k from column k)."""
    weights = np.uint64(1) << np.arange(d, dtype=np.uint64)
    return (bits01.astype(np.uint64) @ weights).astype(_WORD[d])


def _unpack_rows(words: np.ndarray, d: int) -> np.ndarray:
    """row words -> (..., d) uint8 0/1."""
    w = np.asarray(words).astype(np.uint32)
    return ((w[..., None] >> np.arange(d, dtype=np.uint32)) & 1).astype(np.uint8)


# ---------------------------------------------------------------- CSR
class CsrMatrix:
    """Square CSR pattern (``values is None``) or float32-valued matrix.

    Same invariants as the reference (formats.py:96-146): uint32 indices,
    strictly increasing columns per row, no stored exact zeros.  A matrix
    produced on the device (``b2sr_to_csr``, ``from_coo`` of CUDA tensors,
    the R-MAT generator) holds torch CUDA buffers and materialises its host
    arrays lazily.
    """

    __slots__ = ("n", "_row_ptr", "_col_ind", "values", "_nnz", "_dev")

    def __init__(self, n, row_ptr, col_ind, values=None):
        n = int(n)
        if n < 0:
            raise FormatError("matrix dimension must be non-negative")
        rp = _index_array(row_ptr, "row_ptr")
        ci = _index_array(col_ind, "col_ind")
        _check_ptr(rp, n + 1, len(ci), "row_ptr", f"row_ptr must have length n+1 = {n + 1}",
                   "row_ptr[-1] must equal nnz")
        if len(ci) and int(ci.max()) >= n:
            raise FormatError("column index out of range")
        if not _strictly_increasing_in_segments(rp, ci):
            raise FormatError("column indices must be strictly increasing within a row")
        vals = None
        if values is not None:
            vals = np.array(values, dtype=np.float32).reshape(-1) if np.ndim(values) else None
            if vals is None or vals.shape != (len(ci),):
                raise FormatError("values must match nnz")
            if np.any(vals == 0.0):
                raise FormatError("stored values must not be exactly zero")
            vals.flags.writeable = False
        self.n = n
        self._row_ptr, self._col_ind, self.values = rp, ci, vals
        self._nnz = len(ci)
        self._dev = None

    @classmethod
    def _from_device(cls, n: int, row_ptr_t, col_ind_t, nnz: int) -> "CsrMatrix":
        self = cls.__new__(cls)
        self.n = int(n)
        self._row_ptr = self._col_ind = None
        self.values = None
        self._nnz = int(nnz)
        self._dev = (row_ptr_t, col_ind_t)
        return self

    # lazily materialised host arrays
    @property
    def row_ptr(self) -> np.ndarray:
        if self._row_ptr is None:
            a = dev.to_host(self._dev[0], np.uint32, self.n + 1)
            a.flags.writeable = False
            self._row_ptr = a
        return self._row_ptr

    @property
    def col_ind(self) -> np.ndarray:
        if self._col_ind is None:
            a = dev.to_host(self._dev[1], np.uint32, self._nnz)
            a.flags.writeable = False
            self._col_ind = a
        return self._col_ind

    def device_arrays(self):
        """(row_ptr, col_ind) as CUDA byte buffers (uploaded once)."""
        if self._dev is None:
            self._dev = (dev.to_device(self._row_ptr), dev.to_device(self._col_ind))
        return self._dev

    @property
    def nnz(self) -> int:
        return self._nnz

    @property
    def is_pattern(self) -> bool:
        return self.values is None

    @classmethod
    def from_coo(cls, n, rows, cols, values=None) -> "CsrMatrix":
        """Coordinates -> CSR: row-major order, duplicates collapse (last value wins).

        CUDA-tensor coordinates (pattern only) are sorted and de-duplicated
        on the device (radix sort kernel); host arrays take the numpy path.
        """
        n = int(n)
        if dev.is_cuda_tensor(rows) and dev.is_cuda_tensor(cols) and values is None:
            return coo_to_csr_device(n, rows, cols)
        r = np.asarray(rows, dtype=np.int64).reshape(-1)
        c = np.asarray(cols, dtype=np.int64).reshape(-1)
        if r.shape != c.shape:
            raise FormatError("row and column arrays must match")
        if r.size and (min(r.min(), c.min()) < 0 or max(r.max(), c.max()) >= n):
            raise FormatError("coordinate out of range")
        v = None
        if values is not None:
            v = np.asarray(values, dtype=np.float32).reshape(-1)
            if v.shape != r.shape:
                raise FormatError("values must match coordinates")
        key = r * max(n, 1) + c
        order = np.argsort(key, kind="stable")
        key = key[order]
        last = np.ones(len(key), dtype=bool)  # last occurrence of each key
        if len(key) > 1:
            last[:-1] = key[1:] != key[:-1]
        ukey = key[last]
        counts = np.bincount(ukey // max(n, 1), minlength=n) if n else np.zeros(0, np.int64)
        row_ptr = np.concatenate([[0], np.cumsum(counts)]) if n else np.zeros(1, np.int64)
        col = ukey % max(n, 1)
        vals = v[order][last] if v is not None else None
        return cls(n, row_ptr, col, vals)

    def entries(self):
        rows = np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr.astype(np.int64)))
        return rows, self.col_ind.astype(np.int64)

    def row(self, i: int) -> np.ndarray:
        return self.col_ind[int(self.row_ptr[i]): int(self.row_ptr[i + 1])].astype(np.int64)

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.n, self.n))
        r, c = self.entries()
        out[r, c] = 1.0 if self.values is None else self.values
        return out

    def pattern(self) -> "CsrMatrix":
        if self.values is None:
            return self
        return CsrMatrix(self.n, self.row_ptr, self.col_ind)

    def __eq__(self, other):
        if not isinstance(other, CsrMatrix):
            return NotImplemented
        if self.n != other.n or self.nnz != other.nnz:
            return False
        if not (np.array_equal(self.row_ptr, other.row_ptr) and np.array_equal(self.col_ind, other.col_ind)):
            return False
        if (self.values is None) != (other.values is None):
            return False
        return self.values is None or bool(np.array_equal(self.values, other.values))

    __hash__ = None

    def __repr__(self):
        return f"CsrMatrix(n={self.n}, nnz={self.nnz}, pattern={self.is_pattern})"


# ---------------------------------------------------------------- device handle
class _Handle:
    """Owns one ``b2sr_matrix*`` (freed with the Python object)."""

    __slots__ = ("ptr", "n", "dim", "ntr", "num_tiles", "__weakref__")

    def __init__(self, ptr: int):
        self.ptr = ptr
        n, d, ntr, T = ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint32(), ctypes.c_uint64()
        _capi.call("b2sr_info", ptr, ctypes.addressof(n), ctypes.addressof(d), ctypes.addressof(ntr),
                   ctypes.addressof(T))
        self.n, self.dim, self.ntr, self.num_tiles = n.value, d.value, ntr.value, T.value

    def __del__(self):
        if self.ptr and _capi._lib is not None:
            _capi._lib.b2sr_free(self.ptr)
            self.ptr = None


def _new_handle(fn: str, *args) -> _Handle:
    out = ctypes.c_void_p()
    _capi.call(fn, *args, ctypes.byref(out))
    return _Handle(out.value)


# ---------------------------------------------------------------- B2SR
class B2srMatrix:
    """Bit-tile CSR matrix (reference formats.py:228-329).

    ``bit_tiles[t, i]`` is row word ``i`` of stored tile ``t``.
    """

    __slots__ = ("n", "tile_dim", "_trp", "_tci", "_tiles", "_h", "_num_tiles", "_transpose", "_nodiag",
                 "_bfs_push", "_lock", "_dist", "__weakref__")

    def __init__(self, n, tile_dim, tile_row_ptr, tile_col_ind, bit_tiles):
        n = int(n)
        if n <= 0:
            raise FormatError("matrix dimension must be positive")
        td = TileDim.of(tile_dim)
        d, ntr = td.dim, td.tile_rows(n)
        trp = _index_array(tile_row_ptr, "tile_row_ptr")
        tci = _index_array(tile_col_ind, "tile_col_ind")
        T = len(tci)
        _check_ptr(trp, ntr + 1, T, "tile_row_ptr", f"tile_row_ptr must have length {ntr + 1}",
                   "tile_row_ptr[-1] must equal the tile count")
        if T and int(tci.max()) >= ntr:
            raise FormatError("tile column index out of range")
        if not _strictly_increasing_in_segments(trp, tci):
            raise FormatError("tile columns must be strictly increasing within a tile row")
        raw = np.asarray(bit_tiles)
        if raw.dtype.kind not in "ui":
            raise FormatError("bit_tiles must hold unsigned words")
        tiles = np.array(raw, dtype=td.word_dtype, copy=True)
        if tiles.shape != (T, d):
            raise FormatError(f"bit_tiles must have shape ({T}, {d})")
        if T:
            if not tiles.any(axis=1).all():
                raise FormatError("stored tiles must contain at least one set bit")
            if d == 4 and int(tiles.max()) > 0x0F:
                raise FormatError("4-wide tiles must keep the high nibble clear")
            pad = ntr * d - n
            if pad:
                last_row = np.repeat(np.arange(ntr), np.diff(trp.astype(np.int64))) == ntr - 1
                if tiles[last_row, d - pad:].any():
                    raise FormatError("padding bit-rows must be zero")
                keep_cols = (1 << (d - pad)) - 1
                if (tiles[tci == ntr - 1].astype(np.uint64) & np.uint64(~keep_cols & ((1 << d) - 1))).any():
                    raise FormatError("padding bit-columns must be zero")
        tiles.flags.writeable = False
        self.n, self.tile_dim = n, td
        self._trp, self._tci, self._tiles = trp, tci, tiles
        self._h = None
        self._num_tiles = T
        self._transpose = None
        self._nodiag = None
        self._bfs_push = 0  # push-only BFS calls made without a transpose (algorithms.bfs)
        # guards the lazily created device mirror, host arrays and cached
        # transpose / diagonal-free twin: each is created once and never
        # replaced, so a handle read from the matrix stays alive with it
        self._lock = threading.RLock()
        self._dist = None  # per-device-list multi-GPU BFS plans (dist.multi_gpu_bfs)

    @classmethod
    def _wrap(cls, h: _Handle) -> "B2srMatrix":
        """Adopt a device-built matrix (valid by construction)."""
        self = cls.__new__(cls)
        self.n, self.tile_dim = h.n, TileDim(h.dim)
        self._trp = self._tci = self._tiles = None
        self._h = h
        self._num_tiles = h.num_tiles
        self._transpose = None
        self._nodiag = None
        self._bfs_push = 0  # push-only BFS calls made without a transpose (algorithms.bfs)
        # guards the lazily created device mirror, host arrays and cached
        # transpose / diagonal-free twin: each is created once and never
        # replaced, so a handle read from the matrix stays alive with it
        self._lock = threading.RLock()
        self._dist = None  # per-device-list multi-GPU BFS plans (dist.multi_gpu_bfs)
        return self

    # device mirror ---------------------------------------------------
    def handle(self) -> _Handle:
        h = self._h
        if h is None:
            with self._lock:  # two threads' first kernel calls upload once
                if self._h is None:
                    self._h = _new_handle(
                        "b2sr_from_host", self.n, self.dim, self._trp.ctypes.data, self._tci.ctypes.data,
                        self._tiles.ctypes.data, self._num_tiles, dev.stream())
                h = self._h
        return h

    def _materialise(self):
        if self._trp is not None:
            return
        with self._lock:
            if self._trp is None:
                self._download()

    def _download(self):
        h = self._h
        trp = np.zeros(h.ntr + 1, np.uint32)
        tci = np.zeros(h.num_tiles, np.uint32)
        tiles = np.zeros((h.num_tiles, self.dim), self.tile_dim.word_dtype)
        _capi.call("b2sr_to_host", h.ptr, trp.ctypes.data, tci.ctypes.data, tiles.ctypes.data, dev.stream())
        for a in (trp, tci, tiles):
            a.flags.writeable = False
        self._trp, self._tci, self._tiles = trp, tci, tiles

    @property
    def tile_row_ptr(self) -> np.ndarray:
        self._materialise()
        return self._trp

    @property
    def tile_col_ind(self) -> np.ndarray:
        self._materialise()
        return self._tci

    @property
    def bit_tiles(self) -> np.ndarray:
        self._materialise()
        return self._tiles

    @property
    def dim(self) -> int:
        return self.tile_dim.dim

    @property
    def n_tile_rows(self) -> int:
        return self.tile_dim.tile_rows(self.n)

    @property
    def num_tiles(self) -> int:
        return self._num_tiles

    def tile_row_ids(self) -> np.ndarray:
        trp = self.tile_row_ptr.astype(np.int64)
        return np.repeat(np.arange(self.n_tile_rows, dtype=np.int64), np.diff(trp))

    @property
    def nnz(self) -> int:
        if not self._num_tiles:
            return 0
        if self._tiles is not None:
            return int(np.bitwise_count(self._tiles).sum())
        rp = dev.empty_bytes(4 * (self.n + 1))
        nnz = ctypes.c_uint64()
        _capi.call("b2sr_to_csr_rowptr", self.handle().ptr, dev.ptr(rp), ctypes.addressof(nnz), dev.stream())
        return int(nnz.value)

    def __eq__(self, other):
        if not isinstance(other, B2srMatrix):
            return NotImplemented
        if self.n != other.n or self.dim != other.dim or self.num_tiles != other.num_tiles:
            return False
        if self._h is not None and other._h is not None:
            eq = ctypes.c_int()
            _capi.call("b2sr_equal", self._h.ptr, other._h.ptr, dev.stream(), ctypes.addressof(eq))
            return bool(eq.value)
        return (np.array_equal(self.tile_row_ptr, other.tile_row_ptr)
                and np.array_equal(self.tile_col_ind, other.tile_col_ind)
                and np.array_equal(self.bit_tiles, other.bit_tiles))

    __hash__ = None

    def __repr__(self):
        return f"B2srMatrix(n={self.n}, dim={self.dim}, tiles={self.num_tiles})"


# ---------------------------------------------------------------- BitVector
def _valid_mask(n: int, td: TileDim) -> np.ndarray:
    d, nw = td.dim, td.tile_rows(n)
    m = np.full(nw, (1 << d) - 1, dtype=np.uint64)
    if nw and n % d:
        m[-1] = (1 << (n % d)) - 1
    return m.astype(td.word_dtype)


class BitVector:
    """Length-n bits in tile-word layout (reference formats.py:332-441)."""

    __slots__ = ("n", "tile_dim", "words")

    def __init__(self, n: int, tile_dim, words=None):
        n = int(n)
        if n < 0:
            raise FormatError("vector length must be non-negative")
        td = TileDim.of(tile_dim)
        nw = td.tile_rows(n)
        if words is None:
            w = np.zeros(nw, dtype=td.word_dtype)
        else:
            w = np.array(words, dtype=td.word_dtype).reshape(np.shape(words))
            if w.shape != (nw,):
                raise FormatError(f"expected {nw} words, got shape {w.shape}")
            w &= _valid_mask(n, td)
        w.flags.writeable = False
        self.n, self.tile_dim, self.words = n, td, w

    @classmethod
    def zeros(cls, n: int, tile_dim) -> "BitVector":
        return cls(n, tile_dim)

    @classmethod
    def from_bools(cls, flags, tile_dim) -> "BitVector":
        f = np.asarray(flags, dtype=bool).reshape(-1)
        td = TileDim.of(tile_dim)
        padded = np.zeros(td.tile_rows(len(f)) * td.dim, dtype=np.uint8)
        padded[: len(f)] = f
        return cls(len(f), td, _pack_rows(padded.reshape(-1, td.dim), td.dim))

    @classmethod
    def from_indices(cls, n: int, indices, tile_dim) -> "BitVector":
        idx = np.asarray(indices, dtype=np.int64).reshape(-1)
        if idx.size and (idx.min() < 0 or idx.max() >= n):
            raise FormatError("bit index out of range")
        f = np.zeros(int(n), dtype=bool)
        f[idx] = True
        return cls.from_bools(f, tile_dim)

    @property
    def dim(self) -> int:
        return self.tile_dim.dim

    def to_bools(self) -> np.ndarray:
        return _unpack_rows(self.words, self.dim).reshape(-1)[: self.n].astype(bool)

    def to_indices(self) -> np.ndarray:
        return np.flatnonzero(self.to_bools())

    def get(self, i: int) -> bool:
        if not 0 <= i < self.n:
            raise IndexError(f"bit {i} out of range for length {self.n}")
        return bool((int(self.words[i // self.dim]) >> (i % self.dim)) & 1)

    def count(self) -> int:
        return int(np.bitwise_count(self.words).sum()) if len(self.words) else 0

    def any(self) -> bool:
        return bool(self.words.any())

    def invert(self) -> "BitVector":
        return BitVector(self.n, self.tile_dim, ~self.words)

    def _same(self, other):
        if not isinstance(other, BitVector):
            raise TypeError("expected a BitVector")
        if self.n != other.n or self.dim != other.dim:
            raise ValueError("bit vectors must share length and tile width")

    def __or__(self, other):
        self._same(other)
        return BitVector(self.n, self.tile_dim, self.words | other.words)

    def __and__(self, other):
        self._same(other)
        return BitVector(self.n, self.tile_dim, self.words & other.words)

    def repack(self, tile_dim) -> "BitVector":
        return BitVector.from_bools(self.to_bools(), tile_dim)

    def __eq__(self, other):
        if not isinstance(other, BitVector):
            return NotImplemented
        return self.n == other.n and self.dim == other.dim and bool(np.array_equal(self.words, other.words))

    __hash__ = None

    def __repr__(self):
        return f"BitVector(n={self.n}, dim={self.dim}, set={self.count()})"


# ---------------------------------------------------------------- conversions (device)
def coo_to_csr_device(n: int, rows, cols, symmetrize=False, drop_loops=False) -> CsrMatrix:
    """Device COO -> CSR (radix sort + unique), rows/cols uint32-compatible CUDA tensors."""
    t = dev.torch()
    r = rows.to(t.int32).contiguous()
    c = cols.to(t.int32).contiguous()
    if r.numel() != c.numel():
        raise FormatError("row and column arrays must match")
    m = r.numel()
    if m and (int(t.minimum(r.min(), c.min())) < 0 or int(t.maximum(r.max(), c.max())) >= n):
        raise FormatError("coordinate out of range")
    rp = dev.empty_bytes(4 * (n + 1))
    ci = dev.empty_bytes(4 * max(1, (2 * m if symmetrize else m)))
    nnz = ctypes.c_uint64()
    _capi.call("b2sr_coo_to_csr", n, m, r.data_ptr(), c.data_ptr(), int(symmetrize), int(drop_loops),
               dev.ptr(rp), dev.ptr(ci), ctypes.addressof(nnz), dev.stream())
    return CsrMatrix._from_device(n, rp, ci, nnz.value)


def csr_to_b2sr(csr: CsrMatrix, tile_dim) -> B2srMatrix:
    """CSR pattern -> B2SR on the device (K1 count/scan + K2 merge/pack kernels).

    Values are ignored, as in the reference (formats.py:444-464).
    """
    td = TileDim.of(tile_dim)
    if csr.n == 0:
        raise FormatError("cannot tile an empty matrix")
    rp, ci = csr.device_arrays()
    h = _new_handle("b2sr_from_csr", csr.n, td.dim, dev.ptr(rp), dev.ptr(ci), csr.nnz, dev.stream())
    return B2srMatrix._wrap(h)


def b2sr_to_csr(m: B2srMatrix) -> CsrMatrix:
    """Expand tiles back to a CSR pattern on the device (formats.py:467-474)."""
    h = m.handle()
    rp = dev.empty_bytes(4 * (m.n + 1))
    nnz = ctypes.c_uint64()
    _capi.call("b2sr_to_csr_rowptr", h.ptr, dev.ptr(rp), ctypes.addressof(nnz), dev.stream())
    ci = dev.empty_bytes(4 * max(1, nnz.value))
    _capi.call("b2sr_to_csr_fill", h.ptr, dev.ptr(rp), dev.ptr(ci), dev.stream())
    return CsrMatrix._from_device(m.n, rp, ci, nnz.value)


def b2sr_transpose(m: B2srMatrix) -> B2srMatrix:
    """Tile-form transpose on the device (K3; formats.py:477-489).

    Matrices are immutable, so the result is cached on ``m`` (and ``m`` on
    the result): repeated ``bfs``/``sssp`` calls transpose once.
    """
    def cached():
        c = m._transpose
        return c() if isinstance(c, weakref.ref) else c

    t = cached()
    if t is not None:
        return t
    with m._lock:
        t = cached()
        if t is None:
            h = m.handle()
            t = B2srMatrix._wrap(_new_handle("b2sr_transpose", h.ptr, dev.stream()))
            t._transpose = weakref.ref(m)  # no reference cycle: device memory is freed by refcounting
            m._transpose = t
    return t


def drop_diagonal(m: B2srMatrix) -> B2srMatrix:
    """csr_to_b2sr(_drop_diagonal(b2sr_to_csr(m))) done in tile form (algorithms.py:96-101, 111).
    Matrices are immutable, so the result is cached on ``m`` (as transposes are)."""
    if m._nodiag is None:
        with m._lock:
            if m._nodiag is None:
                h = m.handle()
                m._nodiag = B2srMatrix._wrap(_new_handle("b2sr_drop_diagonal", h.ptr, dev.stream()))
    return m._nodiag


# ---------------------------------------------------------------- byte accounting
def storage_bytes(m: B2srMatrix) -> int:
    """4-byte tile indices plus tile payload (formats.py:492-494)."""
    return 4 * (m.n_tile_rows + 1) + 4 * m.num_tiles + m.num_tiles * m.tile_dim.tile_bytes


def csr_storage_bytes(csr: CsrMatrix) -> int:
    """CSR with 4-byte indices and 4-byte values, values counted for patterns too."""
    return 4 * (csr.n + 1) + 8 * csr.nnz


def compression_ratio(m: B2srMatrix, csr: CsrMatrix) -> float:
    return storage_bytes(m) / csr_storage_bytes(csr)


def nonzero_density(csr: CsrMatrix) -> float:
    if csr.n == 0:
        raise ValueError("density of an empty matrix is undefined")
    return csr.nnz / float(csr.n) ** 2


# ---------------------------------------------------------------- container
def save_b2sr(m: B2srMatrix, path) -> None:
    """Little-endian container (formats.py:517-531): 28-byte header then the
    three raw arrays.  A device-resident matrix is written straight from HBM
    (one D2H per array into page-locked memory) without materialising -- and
    caching -- host copies on the matrix."""
    with open(path, "wb") as fh:
        fh.write(_HEADER.pack(_MAGIC, _VERSION, m.n, m.dim, m.n_tile_rows, m.num_tiles))
        if m._trp is not None:
            fh.write(np.ascontiguousarray(m._trp, "<u4").tobytes())
            fh.write(np.ascontiguousarray(m._tci, "<u4").tobytes())
            fh.write(np.ascontiguousarray(m._tiles, m.tile_dim.word_dtype).tobytes())
            return
        h = m.handle()
        t = dev.torch()
        sizes = (4 * (h.ntr + 1), 4 * m.num_tiles, m.num_tiles * m.dim * m.tile_dim.word_dtype.itemsize)
        bufs = [t.empty(max(b, 1), dtype=t.uint8, pin_memory=True) for b in sizes]
        _capi.call("b2sr_to_host", h.ptr, bufs[0].data_ptr(), bufs[1].data_ptr(), bufs[2].data_ptr(), dev.stream())
        for b, nbytes in zip(bufs, sizes):
            if nbytes:
                fh.write(memoryview(b.numpy()[:nbytes]))


def load_b2sr(path) -> B2srMatrix:
    """Read a container written by save_b2sr (formats.py:533-554).  The header
    and size checks run on the host (same FormatError cases and messages);
    the arrays go straight from the file buffer to HBM and the tile
    invariants of formats.py:242-295 are checked there (b2sr_from_host_checked)
    -- no O(T*d) host pass.  The returned matrix keeps read-only host views
    of the file buffer, so touching its arrays costs no copy back."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < _HEADER.size:
        raise FormatError("container truncated before header end")
    magic, version, n, dim, ntr, T = _HEADER.unpack_from(raw)
    if magic != _MAGIC:
        raise FormatError("bad magic; not a tile-matrix container")
    if version != _VERSION:
        raise FormatError(f"unsupported container version {version}")
    if dim not in TILE_DIMS:
        raise FormatError(f"unsupported tile dim {dim}")
    td = TileDim(dim)
    if n <= 0 or ntr != td.tile_rows(n):
        raise FormatError("inconsistent header dimensions")
    want = _HEADER.size + 4 * (ntr + 1) + 4 * T + T * td.tile_bytes
    if len(raw) != want:
        raise FormatError(f"container size {len(raw)} does not match header ({want} expected)")
    o = _HEADER.size
    trp = np.frombuffer(raw, "<u4", ntr + 1, o)
    o += 4 * (ntr + 1)
    tci = np.frombuffer(raw, "<u4", T, o)
    o += 4 * T
    tiles = np.frombuffer(raw, td.word_dtype, T * dim, o).reshape(T, dim)
    h = _new_handle("b2sr_from_host_checked", n, dim, trp.ctypes.data, tci.ctypes.data, tiles.ctypes.data, T,
                    dev.stream())
    m = B2srMatrix._wrap(h)
    m._trp, m._tci, m._tiles = trp, tci, tiles  # read-only views of the file buffer
    return m
