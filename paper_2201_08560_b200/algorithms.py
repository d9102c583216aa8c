"""Graph algorithms as device-resident semiring loops (drop-in for b2sr/algorithms.py).

Each driver keeps its per-sweep state in HBM and runs the loop natively in
libb2sr_sm100.so (csrc/drivers.cu); Python only validates arguments, owns
buffers and turns the final vector into the reference's ``AlgoResult``.

=====================  ===========================================  =================
reference              B200 path                                    parity
=====================  ===========================================  =================
bfs :75-93             push-only levels over a until transposed;    bit-exact levels,
                       then K3 + direction-optimizing push/pull     same iterations
sssp :104-124          BFS levels (= unit-weight distances); or     bit-exact, same
                       diagonal drop + K3 + min-plus(1) rounds      iterations
pagerank :127-163      K6 arithmetic (ascending-j order) + fused    bit-exact ranks and
                       update + numpy-exact pairwise delta          iterations
connected_components   K6 min-plus(0) + parallel hook/shortcut      bit-exact labels;
:166-196                                                            sweep count may
                                                                    differ (parallel
                                                                    hooking)
triangle_count         lower triangle + K1/K2 + K8 with B=L         exact count
:199-215
=====================  ===========================================  =================
"""

from __future__ import annotations

import ctypes
import os
import weakref
from dataclasses import dataclass

import numpy as np

from . import _capi
from . import _device as dev
from .errors import FormatError
from .formats import B2srMatrix, CsrMatrix, b2sr_transpose, csr_to_b2sr, drop_diagonal
from .kernels import resolve_workers


@dataclass(frozen=True)
class AlgoParams:
    """Iteration controls (PageRank uses all three)."""

    alpha: float = 0.85
    epsilon: float = 1e-9
    max_iter: int = 10

    def __post_init__(self):
        if not 0.0 < self.alpha < 1.0:
            raise ValueError("alpha must lie strictly between 0 and 1")
        if self.epsilon <= 0.0:
            raise ValueError("epsilon must be positive")
        if self.max_iter < 1:
            raise ValueError("max_iter must be at least 1")


@dataclass(frozen=True)
class AlgoResult:
    per_vertex: np.ndarray | None
    iterations: int
    converged: bool
    count: int | None = None

    def to_report(self) -> dict:
        doc = {"kind": "run", "iterations": self.iterations, "converged": self.converged}
        if self.count is not None:
            doc["count"] = self.count
        if self.per_vertex is not None:
            doc["perVertex"] = ["inf" if np.isinf(v) else v for v in self.per_vertex.tolist()]
        return doc


def _source(n: int, src) -> int:
    src = int(src)
    if not 0 <= src < n:
        raise ValueError(f"source vertex {src} out of range for n={n}")
    return src


# BFS calls on a matrix without a transpose that run push-only before the
# transpose is built: the transpose (K3 + pull plans) costs about as much as a
# dozen push-only traversals and saves ~half of each later one (ski rental).
BFS_PUSH_CALLS = int(os.environ.get("B2SR_BFS_PUSH_CALLS", "8"))


def _cached_transpose(a: B2srMatrix):
    t = a._transpose
    return t() if isinstance(t, weakref.ref) else t


def bfs(a: B2srMatrix, src: int, *, workers: int | None = None, devices=None) -> AlgoResult:
    """Level-synchronous BFS; hop counts, +inf where unreachable.

    The reference transposes on every call (algorithms.py:78).  Here the
    transpose is cached on the matrix; until one exists (and for the first
    BFS_PUSH_CALLS calls) d = 4/8 matrices run push-only levels over ``a``,
    which need no transpose at all.  Levels and iterations are identical.

    ``devices`` (or env B2SR_GPUS): spread the traversal over several GPUs
    from this process -- a's and at's tile rows cut into blocks, one rank per
    GPU, NCCL between them (dist.multi_gpu_bfs, b2sr_dist_bfs_*; d = 4, 8).
    Same levels and iterations.  ``workers`` stays the reference's thread
    count knob (validated, results independent of it).
    """
    src = _source(a.n, src)
    resolve_workers(workers)
    from . import dist

    devs = dist.resolve_devices(devices)
    if len(devs) > 1:
        if a.dim > 8:
            raise ValueError("multi-GPU bfs supports tile dims 4 and 8")
        at = _cached_transpose(a)
        at = at if at is not None else b2sr_transpose(a)
        lv, it = dist.multi_gpu_bfs(a, at, src, devs)
        return AlgoResult(per_vertex=lv, iterations=int(it), converged=True)
    levels = dev.empty_bytes(8 * a.n)
    it = ctypes.c_int64()
    at = _cached_transpose(a)
    if at is None and a.dim <= 8 and a._bfs_push < BFS_PUSH_CALLS:
        a._bfs_push += 1
        _capi.call("b2sr_bfs", a.handle().ptr, None, src, dev.ptr(levels), ctypes.addressof(it), dev.stream())
        return AlgoResult(per_vertex=dev.to_host(levels, np.float64, a.n), iterations=int(it.value), converged=True)
    at = at if at is not None else b2sr_transpose(a)
    _capi.call("b2sr_bfs", a.handle().ptr, at.handle().ptr, src, dev.ptr(levels), ctypes.addressof(it), dev.stream())
    return AlgoResult(per_vertex=dev.to_host(levels, np.float64, a.n), iterations=int(it.value), converged=True)


def sssp(a: B2srMatrix, src: int, *, workers: int | None = None) -> AlgoResult:
    """Unit-weight shortest paths (algorithms.py:104-124).

    The reference relaxes ``dist = min(dist, bff(at, dist, min_plus(1)))``
    until a round changes nothing (at most n-1 rounds).  With unit weights
    round k settles exactly the vertices at hop distance k, so the result is
    the BFS level vector (self-loops never shorten a path) and the round count
    is min(BFS sweeps, n-1): the BFS driver computes the same bits at BFS
    cost.  ``B2SR_SSSP=relax`` runs the min-plus relaxation driver instead
    (tests check both against the reference's vectors).
    """
    src = _source(a.n, src)
    resolve_workers(workers)
    if os.environ.get("B2SR_SSSP", "bfs") == "relax":
        return _sssp_relax(a, src)
    r = bfs(a, src)
    return AlgoResult(per_vertex=r.per_vertex, iterations=min(r.iterations, a.n - 1), converged=True)


def _sssp_relax(a: B2srMatrix, src: int) -> AlgoResult:
    """The reference's loop on the device: drop the diagonal, transpose, then
    K6 min-plus(1) rounds with a fused np.minimum / changed flag."""
    at = b2sr_transpose(drop_diagonal(a))
    dist = dev.empty_bytes(8 * a.n)
    it = ctypes.c_int64()
    _capi.call("b2sr_sssp", at.handle().ptr, src, dev.ptr(dist), ctypes.addressof(it), dev.stream())
    return AlgoResult(per_vertex=dev.to_host(dist, np.float64, a.n), iterations=int(it.value), converged=True)


def pagerank(a: B2srMatrix, out_degree, params: AlgoParams | None = None, *,
             workers: int | None = None) -> AlgoResult:
    """Damped power iteration; ``a`` is the TRANSPOSED adjacency (a[i,j]=1 for j->i)."""
    params = params or AlgoParams()
    deg = np.asarray(out_degree, dtype=np.float64).reshape(-1)
    if deg.shape != (a.n,):
        raise ValueError(f"expected a length-{a.n} out-degree vector")
    resolve_workers(workers)
    dd = dev.to_device(deg)
    rank = dev.empty_bytes(8 * a.n)
    it, conv, bad = ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64(-1)
    _capi.call("b2sr_pagerank", a.handle().ptr, dev.ptr(dd), float(params.alpha), float(params.epsilon),
               int(params.max_iter), dev.ptr(rank), ctypes.addressof(it), ctypes.addressof(conv),
               ctypes.addressof(bad), dev.stream())
    return AlgoResult(per_vertex=dev.to_host(rank, np.float64, a.n), iterations=int(it.value),
                      converged=bool(conv.value))


def connected_components(a: B2srMatrix, *, workers: int | None = None) -> AlgoResult:
    """Min-id component labels of a symmetric pattern."""
    if a != b2sr_transpose(a):
        raise FormatError("connected components requires a symmetric pattern")
    resolve_workers(workers)
    labels = dev.empty_bytes(8 * a.n)
    it = ctypes.c_int64()
    _capi.call("b2sr_cc", a.handle().ptr, dev.ptr(labels), ctypes.addressof(it), dev.stream())
    return AlgoResult(per_vertex=dev.to_host(labels, np.float64, a.n), iterations=int(it.value), converged=True)


def lower_triangle(csr: CsrMatrix) -> CsrMatrix:
    """Strictly-below-diagonal part of a pattern, computed on the device."""
    n = csr.n
    rp, ci = csr.device_arrays()
    lrp = dev.empty_bytes(4 * (n + 1))
    lnnz = ctypes.c_uint64()
    _capi.call("b2sr_csr_lower_rowptr", n, dev.ptr(rp), dev.ptr(ci), dev.ptr(lrp), ctypes.addressof(lnnz),
               dev.stream())
    lci = dev.empty_bytes(4 * max(1, lnnz.value))
    _capi.call("b2sr_csr_lower_fill", n, dev.ptr(rp), dev.ptr(ci), dev.ptr(lrp), dev.ptr(lci), dev.stream())
    return CsrMatrix._from_device(n, lrp, lci, lnnz.value)


def _degree_oriented(csr: CsrMatrix) -> CsrMatrix:
    """Edges (u, v) with (deg u, u) < (deg v, v) of a symmetric pattern (device).
    Triangle counting uses it in place of the ID-ordered lower triangle: the
    count sum_{(i,j) in L} (L L^T)_ij is the same for any total vertex order."""
    n = csr.n
    rp, ci = csr.device_arrays()
    orp = dev.empty_bytes(4 * (n + 1))
    onnz = ctypes.c_uint64()
    _capi.call("b2sr_csr_orient_rowptr", n, dev.ptr(rp), dev.ptr(ci), dev.ptr(orp), ctypes.addressof(onnz),
               dev.stream())
    oci = dev.empty_bytes(4 * max(1, onnz.value))
    _capi.call("b2sr_csr_orient_fill", n, dev.ptr(rp), dev.ptr(ci), dev.ptr(orp), dev.ptr(oci), dev.stream())
    return CsrMatrix._from_device(n, orp, oci, onnz.value)


def _tc_count(lower_b2sr: B2srMatrix) -> int:
    out = ctypes.c_int64()
    _capi.call("b2sr_tc", lower_b2sr.handle().ptr, ctypes.addressof(out), dev.stream())
    return int(out.value)


def triangle_count(csr: CsrMatrix, tile_dim, *, workers: int | None = None) -> AlgoResult:
    """Triangles of an undirected simple graph: sum over L of (L @ L^T)."""
    pattern = csr.pattern()
    resolve_workers(workers)
    full = csr_to_b2sr(pattern, tile_dim)
    if full.nnz != drop_diagonal(full).nnz:
        raise FormatError("triangle counting requires a loop-free pattern")
    if full != b2sr_transpose(full):
        raise FormatError("triangle counting requires a symmetric pattern")
    # the masked SpGEMM runs on the degree-oriented DAG (edges towards higher
    # degree): the same count as the reference's ID-ordered lower triangle,
    # with every intersected tile row short (R-MAT s20 d=4: 25.8 vs 34 ms).
    # B2SR_TC_ORIENT=id restores the lower triangle (A/B).
    orient = os.environ.get("B2SR_TC_ORIENT", "degree") != "id"
    lo = csr_to_b2sr(_degree_oriented(pattern) if orient else lower_triangle(pattern), tile_dim)
    return AlgoResult(per_vertex=None, iterations=1, converged=True, count=_tc_count(lo))
