"""ctypes front end of the C oracle (oracle/b2sr_oracle.c) -- TEST INFRASTRUCTURE.

The C file restates the reference algorithms of ``b2sr`` 0.1.0 (citations
per function there).  This module gives them numpy-array signatures that
mirror the reference API so parity tests read like the reference's own.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module; the product package never does.

Matrices are passed around as plain tuples ``(n, d, trp, tci, tiles)`` with
the reference's array layout (formats.py:228-240): ``trp`` uint32[ntr+1],
``tci`` uint32[T], ``tiles`` word[T, d] (uint8/uint8/uint16/uint32).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "liboracle.so"
_WORD = {4: np.uint8, 8: np.uint8, 16: np.uint16, 32: np.uint32}

RING_ID = {"boolean": 0, "arithmetic": 1, "minplus": 2, "maxtimes": 3}


def build() -> Path:
    """Compile liboracle.so with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        _lib = ctypes.CDLL(str(_LIB_PATH))
        _declare(_lib)
    return _lib


def _declare(L):
    P = ctypes.c_void_p
    u32, i32, u64, i64, f64 = (ctypes.c_uint32, ctypes.c_int, ctypes.c_uint64,
                               ctypes.c_int64, ctypes.c_double)
    sig = {
        "orc_max_threads": (i32, []),
        "orc_csr_to_b2sr_count": (i64, [u32, i32, P, P, P, i32]),
        "orc_csr_to_b2sr_fill": (None, [u32, i32, P, P, P, P, P, i32]),
        "orc_b2sr_transpose": (None, [u32, i32, P, P, P, P, P, P]),
        "orc_b2sr_to_csr": (u64, [u32, i32, P, P, P, P, P]),
        "orc_used_columns": (None, [u32, i32, P, P, P, P]),
        "orc_bmv_bbb": (None, [u32, i32, P, P, P, P, P, P, i32]),
        "orc_bmv_bbf": (None, [u32, i32, P, P, P, P, P, P, i32]),
        "orc_bmv_bff": (i32, [u32, i32, P, P, P, P, i32, f64, P, P, P, P, i32]),
        "orc_bmm_sum": (i64, [u32, i32, P, P, P, P, P, P, i32]),
        "orc_bmm_sum_masked": (i64, [u32, i32, P, P, P, P, P, P, P, P, P, i32]),
        "orc_pairwise_sum": (f64, [P, i64]),
        "orc_bfs": (i64, [u32, i32, P, P, P, u32, P, i32]),
        "orc_sssp": (i64, [u32, i32, P, P, P, u32, P, i32]),
        "orc_pagerank": (i64, [u32, i32, P, P, P, P, f64, f64, i64, P, P, P, i32]),
        "orc_cc": (i64, [u32, i32, P, P, P, P, i32]),
        "orc_rmat_edges": (None, [i32, u64, u64, P, P]),
        "orc_coo_to_csr": (u64, [u32, u64, P, P, i32, i32, P, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


def _p(a):
    return None if a is None else a.ctypes.data


def _workers(workers):
    return int(workers) if workers else os.cpu_count() or 1


def word_dtype(d):
    return np.dtype(_WORD[d])


def tile_rows(n, d):
    return -(-n // d)


# --------------------------------------------------------------- formats
def csr_to_b2sr(n, row_ptr, col_ind, d, workers=None):
    """formats.py:444-464.  Returns (n, d, trp, tci, tiles)."""
    row_ptr = np.ascontiguousarray(row_ptr, np.uint32)
    col_ind = np.ascontiguousarray(col_ind, np.uint32)
    ntr = tile_rows(n, d)
    trp = np.zeros(ntr + 1, np.uint32)
    T = lib().orc_csr_to_b2sr_count(n, d, _p(row_ptr), _p(col_ind), _p(trp), _workers(workers))
    if T > 0xFFFFFFFF:
        raise OverflowError("tile count exceeds 32-bit index range")
    tci = np.zeros(T, np.uint32)
    tiles = np.zeros((T, d), _WORD[d])
    lib().orc_csr_to_b2sr_fill(n, d, _p(row_ptr), _p(col_ind), _p(trp), _p(tci), _p(tiles),
                               _workers(workers))
    return (n, d, trp, tci, tiles)


def transpose(m):
    """formats.py:477-489."""
    n, d, trp, tci, tiles = m
    T = len(tci)
    trp2 = np.zeros_like(trp)
    tci2 = np.zeros(T, np.uint32)
    tiles2 = np.zeros((T, d), _WORD[d])
    lib().orc_b2sr_transpose(n, d, _p(trp), _p(tci), _p(np.ascontiguousarray(tiles)),
                             _p(trp2), _p(tci2), _p(tiles2))
    return (n, d, trp2, tci2, tiles2)


def b2sr_to_csr(m):
    """formats.py:467-474.  Returns (row_ptr, col_ind)."""
    n, d, trp, tci, tiles = m
    tiles = np.ascontiguousarray(tiles)
    row_ptr = np.zeros(n + 1, np.uint32)
    nnz = lib().orc_b2sr_to_csr(n, d, _p(trp), _p(tci), _p(tiles), _p(row_ptr), None)
    col_ind = np.zeros(nnz, np.uint32)
    lib().orc_b2sr_to_csr(n, d, _p(trp), _p(tci), _p(tiles), _p(row_ptr), _p(col_ind))
    return row_ptr, col_ind


def used_columns(m):
    """kernels.py:86-94."""
    n, d, trp, tci, tiles = m
    out = np.zeros(n, np.uint8)
    lib().orc_used_columns(n, d, _p(trp), _p(tci), _p(np.ascontiguousarray(tiles)), _p(out))
    return out.astype(bool)


# --------------------------------------------------------------- vectors
def pack_bits(flags, d):
    """Bools -> tile-word BitVector layout (formats.py:332-370)."""
    flags = np.asarray(flags, bool).ravel()
    n = len(flags)
    ntr = tile_rows(n, d)
    pad = np.zeros(ntr * d, np.uint64)
    pad[:n] = flags
    w = (pad.reshape(ntr, d) << np.arange(d, dtype=np.uint64)).sum(axis=1)
    return w.astype(_WORD[d])


def unpack_bits(words, n, d):
    w = np.asarray(words).astype(np.uint64)
    bits = (w[:, None] >> np.arange(d, dtype=np.uint64)) & np.uint64(1)
    return bits.reshape(-1)[:n].astype(bool)


# --------------------------------------------------------------- kernels
def bmv_bbb(m, x_words, keep_words=None, workers=None):
    """kernels.py:97-115 / 219-225.  Returns y words."""
    n, d, trp, tci, tiles = m
    y = np.zeros(tile_rows(n, d), _WORD[d])
    x_words = np.ascontiguousarray(x_words, _WORD[d])
    kw = None if keep_words is None else np.ascontiguousarray(keep_words, _WORD[d])
    lib().orc_bmv_bbb(n, d, _p(trp), _p(tci), _p(np.ascontiguousarray(tiles)), _p(x_words), _p(kw),
                      _p(y), _workers(workers))
    return y


def bmv_bbf(m, x_words, keep_words=None, workers=None):
    """kernels.py:118-137 / 228-234.  Returns float64[n]."""
    n, d, trp, tci, tiles = m
    y = np.zeros(n, np.float64)
    x_words = np.ascontiguousarray(x_words, _WORD[d])
    kw = None if keep_words is None else np.ascontiguousarray(keep_words, _WORD[d])
    lib().orc_bmv_bbf(n, d, _p(trp), _p(tci), _p(np.ascontiguousarray(tiles)), _p(x_words), _p(kw),
                      _p(y), _workers(workers))
    return y


class OracleError(ValueError):
    pass


def bmv_bff(m, x, ring, inc=0.0, scale=None, keep_words=None, workers=None):
    """kernels.py:140-216 / 237-249.  ring in {'arithmetic','minplus','maxtimes'}."""
    n, d, trp, tci, tiles = m
    x = np.ascontiguousarray(x, np.float64)
    sc = None if scale is None else np.ascontiguousarray(scale, np.float64)
    kw = None if keep_words is None else np.ascontiguousarray(keep_words, _WORD[d])
    y = np.zeros(n, np.float64)
    bad = ctypes.c_int64(-1)
    rc = lib().orc_bmv_bff(n, d, _p(trp), _p(tci), _p(np.ascontiguousarray(tiles)), _p(x),
                           RING_ID[ring], float(inc), _p(sc), _p(kw), _p(y),
                           ctypes.addressof(bad), _workers(workers))
    if rc:
        raise OracleError({1: "boolean ring", 2: "scale with non-arithmetic ring",
                           3: f"zero scale at used column {bad.value}"}[rc])
    return y


def bmm_sum(a, b, workers=None):
    """kernels.py:298-320."""
    n, d = a[0], a[1]
    return int(lib().orc_bmm_sum(n, d, _p(a[2]), _p(a[3]), _p(np.ascontiguousarray(a[4])),
                                 _p(b[2]), _p(b[3]), _p(np.ascontiguousarray(b[4])),
                                 _workers(workers)))


def bmm_sum_masked(a, b, mask, workers=None):
    """kernels.py:323-367."""
    n, d = a[0], a[1]
    return int(lib().orc_bmm_sum_masked(
        n, d, _p(a[2]), _p(a[3]), _p(np.ascontiguousarray(a[4])),
        _p(b[2]), _p(b[3]), _p(np.ascontiguousarray(b[4])),
        _p(mask[2]), _p(mask[3]), _p(np.ascontiguousarray(mask[4])), _workers(workers)))


def pairwise_sum(a):
    a = np.ascontiguousarray(a, np.float64)
    return float(lib().orc_pairwise_sum(_p(a), len(a)))


# --------------------------------------------------------------- drivers
def bfs(m, src, workers=None, symmetric=False):
    """algorithms.py:75-93 (transposes first, as the reference does).  With
    ``symmetric=True`` the caller asserts m == transpose(m) (an undirected
    graph) and the matrix is passed as its own transpose -- the restatement
    rule of SURVEY.md §8c for sizes where the transpose dominates."""
    at = m if symmetric else transpose(m)
    n, d = m[0], m[1]
    levels = np.zeros(n, np.float64)
    it = lib().orc_bfs(n, d, _p(at[2]), _p(at[3]), _p(at[4]), int(src), _p(levels), _workers(workers))
    if it < 0:
        raise RuntimeError("BFS failed to drain its frontier")
    return levels, int(it)


def drop_diagonal_b2sr(m):
    """algorithms.py:96-101 + 111: b2sr_to_csr, drop (i,i), csr_to_b2sr."""
    n, d = m[0], m[1]
    rp, ci = b2sr_to_csr(m)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp.astype(np.int64)))
    keep = rows != ci
    if keep.all():
        return csr_to_b2sr(n, rp, ci, d)
    rows, ci = rows[keep], ci[keep]
    rp2 = np.zeros(n + 1, np.int64)
    np.add.at(rp2, rows + 1, 1)
    return csr_to_b2sr(n, np.cumsum(rp2).astype(np.uint32), ci, d)


def sssp(m, src, workers=None, at=None):
    """algorithms.py:104-124.  ``at`` = transpose(drop_diagonal(m)) when the
    caller already has it (e.g. a loop-free symmetric m is its own)."""
    if at is None:
        at = transpose(drop_diagonal_b2sr(m))
    n, d = m[0], m[1]
    dist = np.zeros(n, np.float64)
    it = lib().orc_sssp(n, d, _p(at[2]), _p(at[3]), _p(at[4]), int(src), _p(dist), _workers(workers))
    return dist, int(it)


def pagerank(a, out_degree, alpha=0.85, epsilon=1e-9, max_iter=10, workers=None):
    """algorithms.py:127-163; ``a`` is the transposed adjacency."""
    n, d = a[0], a[1]
    deg = np.ascontiguousarray(out_degree, np.float64)
    rank = np.zeros(n, np.float64)
    conv = ctypes.c_int(0)
    bad = ctypes.c_int64(-1)
    it = lib().orc_pagerank(n, d, _p(a[2]), _p(a[3]), _p(np.ascontiguousarray(a[4])), _p(deg),
                            float(alpha), float(epsilon), int(max_iter), _p(rank),
                            ctypes.addressof(conv), ctypes.addressof(bad), _workers(workers))
    if it < 0:
        raise OracleError(f"out_degree[{bad.value}] is zero but vertex {bad.value} has out-edges")
    return rank, int(it), bool(conv.value)


def connected_components(m, workers=None):
    """algorithms.py:166-196 (caller guarantees symmetry)."""
    n, d = m[0], m[1]
    labels = np.zeros(n, np.float64)
    it = lib().orc_cc(n, d, _p(m[2]), _p(m[3]), _p(np.ascontiguousarray(m[4])), _p(labels),
                      _workers(workers))
    if it < 0:
        raise RuntimeError("component labels failed to stabilise")
    return labels, int(it)


def lower_triangle(n, row_ptr, col_ind):
    """algorithms.py:218-222."""
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(np.asarray(row_ptr, np.int64)))
    col_ind = np.asarray(col_ind, np.int64)
    keep = rows > col_ind
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows[keep] + 1, 1)
    return np.cumsum(rp).astype(np.uint32), col_ind[keep].astype(np.uint32)


def triangle_count(n, row_ptr, col_ind, d, workers=None):
    """algorithms.py:199-215 (validation done by the caller)."""
    lrp, lci = lower_triangle(n, row_ptr, col_ind)
    lo = csr_to_b2sr(n, lrp, lci, d, workers)
    return bmm_sum_masked(lo, transpose(lo), lo, workers)


# --------------------------------------------------------------- inputs
def rmat_edges(scale, edgefactor=16, seed=1):
    """CPU twin of the device R-MAT generator (csrc/rmat.cu)."""
    m = edgefactor << scale
    src = np.zeros(m, np.uint32)
    dst = np.zeros(m, np.uint32)
    lib().orc_rmat_edges(scale, m, seed, _p(src), _p(dst))
    return src, dst


def coo_to_csr(n, src, dst, symmetrize=False, drop_loops=False):
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    m = len(src)
    row_ptr = np.zeros(n + 1, np.uint32)
    col_ind = np.zeros(2 * m if symmetrize else m, np.uint32)
    nnz = lib().orc_coo_to_csr(n, m, _p(src), _p(dst), int(symmetrize), int(drop_loops),
                               _p(row_ptr), _p(col_ind))
    return row_ptr, col_ind[:nnz].copy()


def rmat_csr(scale, edgefactor=16, seed=1, undirected=True):
    """R-MAT graph as CSR: symmetrized, self-loops dropped, de-duplicated."""
    src, dst = rmat_edges(scale, edgefactor, seed)
    return coo_to_csr(1 << scale, src, dst, symmetrize=undirected, drop_loops=undirected)
