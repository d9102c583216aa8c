"""Row-partitioned multi-GPU drivers (one process per GPU, torch.distributed).

SURVEY.md §8e: the transposed adjacency is cut into contiguous tile-row
blocks, one per rank; every rank keeps the full frontier / visited bit
vectors (n/8 bytes) and its block of the matrix.  Per BFS level:

    sweep   masked pull sweep over the rank's block      (K4 stream: loads of rows
            with unvisited vertices, lazy tile bytes behind sparse frontiers)
    gather  all_gather of the blocks' frontier words    (NCCL over NVLink)
    update  visited |= frontier, levels, any-flag        (k_bfs_update, local)

The blocks have equal tile-row counts, padded to a whole 4-byte word per
rank, so the all-gather output *is* the global frontier -- no compaction.
R-MAT vertices are randomly permuted, so equal row counts balance tiles.
Every rank sees the same gathered frontier, so the termination test needs no
extra collective.  Triangle counting partitions the mask (L) tile rows the
same way, keeps L replicated for the row lookups, and finishes with one
int64 all_reduce.

Results are partition-invariant: the per-row work is identical, only the
owner changes, and the exchange is a pure copy.

The level loop is written against a small ``ops`` interface so the host
logic (partition, exchange, loop, termination) is testable on CPU with the
gloo backend (tests/test_dist_gloo.py plugs in oracle ops); the product ops
are the CUDA kernels below.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from . import _capi
from . import _device as dev
from .formats import B2srMatrix, _Handle, _new_handle


def block_rows(ntr: int, world: int, dim: int) -> int:
    """Tile rows per rank: ceil(ntr / world) rounded up to whole 4-byte words."""
    wb = 4 if dim == 32 else (2 if dim == 16 else 1)
    per_word = 4 // wb
    rows = -(-ntr // world)
    return -(-rows // per_word) * per_word


def partition(ntr: int, world: int, dim: int):
    """[(begin, end)) tile-row ranges, equal padded sizes, clipped to ntr."""
    b = block_rows(ntr, world, dim)
    return [(min(r * b, ntr), min((r + 1) * b, ntr)) for r in range(world)]


class CudaBfsOps:
    """Product ops: the sm_100a kernels through the C ABI."""

    def __init__(self, block: _Handle, n: int, dim: int):
        self.block, self.n, self.dim = block, n, dim

    def buffers(self, global_bytes: int, block_bytes: int):
        return (dev.zeros_bytes(global_bytes), dev.zeros_bytes(global_bytes), dev.zeros_bytes(block_bytes),
                dev.empty_bytes(8 * self.n), dev.zeros_bytes(16))

    def init(self, src, visited, frontier, levels):
        _capi.call("b2sr_bfs_init", self.n, self.dim, src, dev.ptr(visited), dev.ptr(frontier), dev.ptr(levels),
                   dev.stream())

    def sweep(self, frontier, visited, next_block, sparse=False):
        # the block's loads of rows with unvisited vertices only; tile bytes
        # fetched lazily behind a sparse frontier (same output either way)
        flags = 1 | (2 if sparse else 0)  # B2SR_SWEEP_ACTIVE | B2SR_SWEEP_LAZY
        _capi.call("b2sr_bfs_sweep_ex", self.block.ptr, dev.ptr(frontier), dev.ptr(visited), dev.ptr(next_block),
                   flags, dev.stream())

    def update(self, frontier, visited, levels, level, anyflag):
        """visited |= frontier, levels; (any new vertex, frontier vertex count)."""
        anyflag.zero_()
        _capi.call("b2sr_bfs_update_ex", self.n, self.dim, dev.ptr(frontier), dev.ptr(visited), dev.ptr(levels),
                   float(level), dev.ptr(anyflag), dev.ptr(anyflag) + 8, dev.stream())
        h = anyflag.cpu()
        return bool(h[:4].view(dev.torch().int32)[0].item()), int(h[8:16].view(dev.torch().int64)[0].item())

    def levels_to_host(self, levels):
        return dev.to_host(levels, np.float64, self.n)

    def levels_on_device(self, levels):
        return levels.view(dev.torch().float64)[: self.n]


def all_gather_words(dist, out, block, world):
    """Concatenate every rank's block into ``out`` (byte tensors)."""
    if dist.get_backend() == "nccl":
        dist.all_gather_into_tensor(out, block)
    else:  # gloo (CPU tests)
        parts = [out[r * block.numel(): (r + 1) * block.numel()] for r in range(world)]
        tmp = [p.clone() for p in parts]
        dist.all_gather(tmp, block)
        for p, t in zip(parts, tmp):
            p.copy_(t)


class DistributedBfs:
    """BFS over a tile-row-partitioned transposed matrix (one rank per GPU)."""

    def __init__(self, n: int, dim: int, ntr: int, rank: int, world: int, ops, dist):
        self.n, self.dim, self.ntr = n, dim, ntr
        self.rank, self.world, self.ops, self.dist = rank, world, ops, dist
        wb = 4 if dim == 32 else (2 if dim == 16 else 1)
        self.block_bytes = block_rows(ntr, world, dim) * wb
        self.global_bytes = self.block_bytes * world

    @classmethod
    def from_matrix(cls, at: B2srMatrix, dist):
        """Cut this rank's block out of the full transposed matrix on its GPU."""
        rank, world = dist.get_rank(), dist.get_world_size()
        b, e = partition(at.n_tile_rows, world, at.dim)[rank]
        blk = _new_handle("b2sr_row_block", at.handle().ptr, b, e, dev.stream())
        return cls(at.n, at.dim, at.n_tile_rows, rank, world, CudaBfsOps(blk, at.n, at.dim), dist)

    @classmethod
    def from_block(cls, block: _Handle, n: int, dim: int, dist):
        """A rank's own row block (e.g. uploaded with b2sr_block_from_host)."""
        rank, world = dist.get_rank(), dist.get_world_size()
        ntr = -(-n // dim)
        return cls(n, dim, ntr, rank, world, CudaBfsOps(block, n, dim), dist)

    def run(self, src: int, to_host: bool = True):
        """Levels (float64, inf = unreached) and the sweep count; with
        ``to_host=False`` the levels stay on the device (product ops only)."""
        ops = self.ops
        visited, frontier, nxt, levels, anyflag = ops.buffers(self.global_bytes, self.block_bytes)
        ops.init(src, visited, frontier, levels)
        sweeps = 0
        sparse = True  # level 1: the frontier is {src}
        while True:
            ops.sweep(frontier, visited, nxt, sparse)
            all_gather_words(self.dist, frontier, nxt, self.world)
            sweeps += 1
            more, fv = ops.update(frontier, visited, levels, float(sweeps), anyflag)
            sparse = fv * 16 < self.n  # every rank sees the same gathered frontier: same choice
            if sweeps > self.n:
                raise RuntimeError("BFS failed to drain its frontier")
            if not more:
                break
        if not to_host:
            return ops.levels_on_device(levels), sweeps
        return ops.levels_to_host(levels), sweeps


def block_to_host(block: _Handle, pinned: bool = True):
    """(trp, tci, tiles) host copies of a device row block, in pinned memory."""
    t = dev.torch()

    def buf(count, dtype):
        a = t.empty(max(count, 1) * np.dtype(dtype).itemsize, dtype=t.uint8, pin_memory=pinned)
        return a, a.numpy().view(dtype)[:count]

    wdt = {4: np.uint8, 8: np.uint8, 16: np.uint16, 32: np.uint32}[block.dim]
    trp, tci, tiles = buf(block.ntr + 1, np.uint32), buf(block.num_tiles, np.uint32), buf(block.num_tiles * block.dim, wdt)
    _capi.call("b2sr_to_host", block.ptr, trp[1].ctypes.data, tci[1].ctypes.data, tiles[1].ctypes.data, dev.stream())
    t.cuda.synchronize()
    return trp, tci, tiles


def block_from_host(n: int, dim: int, begin: int, end: int, host) -> _Handle:
    """Upload a rank's row block from host arrays (b2sr_block_from_host)."""
    trp, tci, tiles = (h[1] for h in host)
    return _new_handle("b2sr_block_from_host", n, dim, begin, end, trp.ctypes.data, tci.ctypes.data,
                       tiles.ctypes.data, len(tci), dev.stream())


# ---------------------------------------------------------------- native multi-GPU drivers
class Comm:
    """One rank's communicator inside the C library (b2sr_comm_*).

    ``Comm.from_torch(dist)``: NCCL over NVLink / NVSwitch, one process per
    GPU; rank 0 makes the NCCL id and ``torch.distributed`` ships it.
    ``Comm.nccl_single()``: a world of one (same code path, one GPU).
    ``Comm.local(world)``: ``world`` thread-ranks sharing the current GPU
    (the multi-rank level loop testable on one device)."""

    def __init__(self, ptr: int, rank: int, world: int):
        self.ptr, self.rank, self.world = ptr, rank, world

    @classmethod
    def from_torch(cls, dist) -> "Comm":
        rank, world = dist.get_rank(), dist.get_world_size()
        box = [None]
        if rank == 0:
            uid = (ctypes.c_uint8 * 128)()
            _capi.call("b2sr_comm_unique_id", ctypes.addressof(uid))
            box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(box[0])
        out = ctypes.c_void_p()
        _capi.call("b2sr_comm_init", ctypes.addressof(uid), world, rank, ctypes.byref(out))
        return cls(out.value, rank, world)

    @classmethod
    def nccl_single(cls) -> "Comm":
        uid = (ctypes.c_uint8 * 128)()
        _capi.call("b2sr_comm_unique_id", ctypes.addressof(uid))
        out = ctypes.c_void_p()
        _capi.call("b2sr_comm_init", ctypes.addressof(uid), 1, 0, ctypes.byref(out))
        return cls(out.value, 0, 1)

    @classmethod
    def local(cls, world: int) -> list:
        outs = (ctypes.c_void_p * world)()
        _capi.call("b2sr_comm_init_local", world, ctypes.addressof(outs))
        return [cls(outs[r], r, world) for r in range(world)]

    def __del__(self):
        if getattr(self, "ptr", None) and _capi._lib is not None:
            _capi._lib.b2sr_comm_free(self.ptr)
            self.ptr = None


class NativeDistributedBfs:
    """bfs (algorithms.py:75-93) over row blocks of a and at, direction-
    optimizing and device-controlled (b2sr_dist_bfs_*; d = 4, 8): the level
    loop, its exchanges (all-to-all-v of row contributions + all-gather-v of
    the merged rows) and the level plan run in the library on the caller's
    stream, with no host sync per level.  Levels end up on every rank."""

    def __init__(self, comm: Comm, plan: int, n: int, keep=()):
        self.comm, self.plan, self.n = comm, plan, n
        self._keep = keep  # blocks a plan_blocks plan points into

    @classmethod
    def from_matrices(cls, comm: Comm, a: B2srMatrix, at: B2srMatrix) -> "NativeDistributedBfs":
        """Every rank holds the full a and at; the plan cuts its blocks
        (balanced by at's tiles) -- the full matrices may be dropped after."""
        out = ctypes.c_void_p()
        ha, hat = a.handle(), at.handle()
        _capi.call("b2sr_dist_bfs_plan", comm.ptr, ha.ptr, hat.ptr, dev.stream(), ctypes.byref(out))
        return cls(comm, out.value, a.n)

    @classmethod
    def from_blocks(cls, comm: Comm, a_block: _Handle, at_block: _Handle, trp_a, trp_at) -> "NativeDistributedBfs":
        """This rank's blocks (e.g. uploaded with block_from_host) and the
        global tile_row_ptr arrays of a and at (host numpy or device tensors)."""
        def ptr(x):
            return x.data_ptr() if dev.is_cuda_tensor(x) else np.ascontiguousarray(x, np.uint32).ctypes.data

        keep = [np.ascontiguousarray(x, np.uint32) if not dev.is_cuda_tensor(x) else x for x in (trp_a, trp_at)]
        out = ctypes.c_void_p()
        _capi.call("b2sr_dist_bfs_plan_blocks", comm.ptr, a_block.ptr, at_block.ptr, ptr(keep[0]), ptr(keep[1]),
                   dev.stream(), ctypes.byref(out))
        return cls(comm, out.value, a_block.n, keep=(a_block, at_block))

    @property
    def rows(self):
        b, e = ctypes.c_uint32(), ctypes.c_uint32()
        _capi.call("b2sr_dist_bfs_rows", self.plan, ctypes.addressof(b), ctypes.addressof(e))
        return b.value, e.value

    def run(self, src: int, to_host: bool = True, levels=None, stream=None):
        """(levels float64[n], sweeps); ``to_host=False`` keeps the levels on
        the device (a CUDA tensor view)."""
        lv = levels if levels is not None else dev.empty_bytes(8 * self.n)
        it = ctypes.c_int64()
        _capi.call("b2sr_dist_bfs_run", self.plan, int(src), dev.ptr(lv), ctypes.addressof(it),
                   stream if stream is not None else dev.stream())
        if not to_host:
            return lv.view(dev.torch().float64)[: self.n], int(it.value)
        return dev.to_host(lv, np.float64, self.n), int(it.value)

    def __del__(self):
        if getattr(self, "plan", None) and _capi._lib is not None:
            _capi._lib.b2sr_dist_bfs_free(self.plan)
            self.plan = None


def native_triangle_count(comm: Comm, lower: B2srMatrix, stream=None):
    """(count, cuts): the masked SpGEMM of triangle_count with L replicated and
    its mask rows cut by estimated work (b2sr_dist_tc); one int64 all-reduce."""
    out = ctypes.c_int64()
    cuts = (ctypes.c_uint32 * (comm.world + 1))()
    h = lower.handle()
    _capi.call("b2sr_dist_tc", comm.ptr, h.ptr, ctypes.addressof(out), ctypes.addressof(cuts),
               stream if stream is not None else dev.stream())
    return int(out.value), list(cuts)


# ---------------------------------------------------------------- one process, several GPUs
def resolve_devices(devices=None) -> list:
    """The GPUs a drop-in call spreads over: ``devices`` (a count N -> cuda:0..N-1,
    or an explicit list of device ordinals), else env B2SR_GPUS (a count or
    "0,1,..."), else one GPU.  A list may repeat an ordinal: those ranks
    share that GPU (thread-ranks exchanging through device copies -- how the
    multi-rank path is tested on one device)."""
    if devices is None:
        env = os.environ.get("B2SR_GPUS", "").strip()
        if not env:
            return [None]
        devices = [int(x) for x in env.split(",")] if "," in env else int(env)
    if isinstance(devices, (int, np.integer)):
        if devices < 1:
            raise ValueError("devices must be at least 1")
        devices = list(range(int(devices)))
    devices = [int(d) for d in devices]
    if not devices or any(d < 0 for d in devices):
        raise ValueError("devices must be a positive count or a list of device ordinals")
    return devices


def _row_cuts(trp: np.ndarray, world: int, dim: int) -> list:
    """Tile-row blocks balanced by tile count, on 16-byte word boundaries of
    the bit vectors (the rule of b2sr_dist_bfs_plan's k_balanced_cuts)."""
    ntr = len(trp) - 1
    align = 16 // (4 if dim == 32 else 2 if dim == 16 else 1)
    T = int(trp[-1])
    cuts = [0]
    for k in range(1, world):
        r = int(np.searchsorted(trp, T * k // world, side="left"))
        cuts.append(min(ntr, (r + align // 2) // align * align))
    cuts.append(ntr)
    return [max(c, cuts[i - 1]) if i else c for i, c in enumerate(cuts)]


class _MultiGpuBfs:
    """Per-matrix state of bfs(a, src, devices=...): one rank per listed
    device, each holding its rows of a and at (uploaded once from the host
    arrays) and a b2sr_dist_bfs plan; every call runs the ranks' level loops
    concurrently on host threads (the C calls release the GIL)."""

    def __init__(self, a: B2srMatrix, at: B2srMatrix, devs: list):
        t = dev.torch()
        self.n, self.devs = a.n, devs
        world = len(devs)
        trp_a, trp_at = np.ascontiguousarray(a.tile_row_ptr), np.ascontiguousarray(at.tile_row_ptr)
        cuts = _row_cuts(trp_at, world, a.dim)
        host = []
        for mat, trp in ((a, trp_a), (at, trp_at)):
            tci, tiles = mat.tile_col_ind, mat.bit_tiles
            parts = []
            for r in range(world):
                b, e = cuts[r], cuts[r + 1]
                t0, t1 = int(trp[b]), int(trp[e])
                parts.append(((None, (trp[b:e + 1] - trp[b]).astype(np.uint32)), (None, tci[t0:t1]),
                              (None, np.ascontiguousarray(tiles[t0:t1]))))
            host.append(parts)
        if len(set(devs)) == len(devs):  # distinct GPUs: NCCL, ranks initialised together
            uid = (ctypes.c_uint8 * 128)()
            _capi.call("b2sr_comm_unique_id", ctypes.addressof(uid))
            comms = [None] * world
        else:  # repeated ordinals: thread-ranks sharing devices
            t.cuda.set_device(devs[0])
            comms = Comm.local(world)
            uid = None
        self.ranks = [None] * world

        def setup(r):
            t.cuda.set_device(devs[r])
            if uid is not None:
                out = ctypes.c_void_p()
                _capi.call("b2sr_comm_init", ctypes.addressof(uid), world, r, ctypes.byref(out))
                comms[r] = Comm(out.value, r, world)
            b, e = cuts[r], cuts[r + 1]
            ab = block_from_host(a.n, a.dim, b, e, host[0][r])
            atb = block_from_host(a.n, a.dim, b, e, host[1][r])
            self.ranks[r] = NativeDistributedBfs.from_blocks(comms[r], ab, atb, trp_a, trp_at)

        self._each(setup)
        self.cuts = cuts

    def _each(self, fn):
        err, threads = [], []

        def body(r):
            try:
                fn(r)
            except BaseException as e:  # noqa: BLE001 -- re-raised on the caller's thread
                err.append(e)

        for r in range(len(self.devs)):
            threads.append(threading.Thread(target=body, args=(r,)))
            threads[-1].start()
        for th in threads:
            th.join()
        if err:
            raise err[0]

    def run(self, src: int):
        t = dev.torch()
        out = [None] * len(self.devs)

        def go(r):
            t.cuda.set_device(self.devs[r])
            st = t.cuda.Stream()
            with t.cuda.stream(st):
                out[r] = self.ranks[r].run(src, to_host=(r == 0), stream=st.cuda_stream)
                st.synchronize()

        self._each(go)
        return out[0]


_multi_lock = threading.Lock()


def multi_gpu_bfs(a: B2srMatrix, at: B2srMatrix, src: int, devs: list):
    """bfs over several GPUs from one process; plans cached on ``a``."""
    key = tuple(devs)
    with _multi_lock:
        cache = a._dist if a._dist is not None else {}
        a._dist = cache
        state = cache.get(key)
        if state is None:
            state = cache[key] = _MultiGpuBfs(a, at, devs)
    return state.run(src)


# ---------------------------------------------------------------- float-gather drivers
def _slices(n: int, dim: int, world: int, rank: int):
    """(vertex begin, valid count, padded slice length) of this rank's rows."""
    ntr = -(-n // dim)
    b, e = partition(ntr, world, dim)[rank]
    per = block_rows(ntr, world, dim) * dim
    v0 = b * dim
    return b, e, v0, max(0, min(e * dim, n) - v0), per


def _bff_block(blk: _Handle, x, ring: int, inc: float, y):
    bad = ctypes.c_int64(-1)
    _capi.call("b2sr_bmv_bff", blk.ptr, dev.ptr(x), ring, float(inc), None, None, dev.ptr(y),
               ctypes.addressof(bad), dev.stream())


def distributed_pagerank(at: B2srMatrix, out_degree, dist, alpha: float = 0.85, epsilon: float = 1e-9,
                         max_iter: int = 10):
    """PageRank (algorithms.py:127-163) with the tile rows of ``at`` (the
    transposed adjacency) partitioned over ranks.  Per sweep: the rank's rows
    of g = bff(at, rank/deg) and of the update, then one all-gather of the new
    rank/deg slices and one of the |delta| slices; every rank evaluates numpy's
    pairwise delta over the full vector, so the bits and the iteration count
    are those of the single-GPU driver.  Returns (rank, iterations, converged)."""
    t = dev.torch()
    rank, world = dist.get_rank(), dist.get_world_size()
    n, d = at.n, at.dim
    out_degree = np.asarray(out_degree, dtype=np.float64).reshape(-1)
    if out_degree.shape != (n,):
        raise ValueError(f"expected a length-{n} out-degree vector")
    # the check of algorithms.py:143-148 (and of the single-GPU driver): a
    # vertex with out-edges (a used column of the transposed matrix) must not
    # have a zero out-degree -- every rank sees the whole matrix, so every
    # rank raises the same error
    ud = dev.empty_bytes(max(n, 16))
    _capi.call("b2sr_used_columns", at.handle().ptr, dev.ptr(ud), dev.stream())
    used = dev.to_host(ud, np.uint8, n).astype(bool)
    bad = np.flatnonzero(used & (out_degree == 0.0))
    if bad.size:
        j = int(bad[0])
        raise ValueError(f"out_degree[{j}] is zero but vertex {j} has out-edges")
    b, e, v0, cnt, per = _slices(n, d, world, rank)
    blk = _new_handle("b2sr_row_block", at.handle().ptr, b, e, dev.stream())
    full = per * world
    deg = t.zeros(full, dtype=t.float64, device=dev.device())
    deg[:n] = t.as_tensor(np.asarray(out_degree, dtype=np.float64).reshape(-1), device=dev.device())
    r = t.full((full,), 1.0 / n, dtype=t.float64, device=dev.device())
    r[n:] = 0.0
    xs = t.where(deg == 0, t.zeros_like(r), r / t.where(deg == 0, t.ones_like(deg), deg))
    diff = t.zeros(full, dtype=t.float64, device=dev.device())
    g = t.zeros(per + 16, dtype=t.float64, device=dev.device())
    r_loc, xs_loc, diff_loc = (t.zeros(per, dtype=t.float64, device=dev.device()) for _ in range(3))
    out = t.zeros(2, dtype=t.float64, device=dev.device())
    teleport = (1.0 - alpha) / n
    it, conv = 0, False
    while it < max_iter:
        _bff_block(blk, xs, 1, 0.0, g)  # B2SR_RING_ARITHMETIC
        r_loc[:cnt].copy_(r[v0:v0 + cnt])
        _capi.call("b2sr_pr_step", cnt, teleport, float(alpha), dev.ptr(g), dev.ptr(deg[v0:]), dev.ptr(r_loc),
                   dev.ptr(xs_loc), dev.ptr(diff_loc), dev.stream())
        all_gather_words(dist, xs.view(t.uint8), xs_loc.view(t.uint8), world)
        all_gather_words(dist, diff.view(t.uint8), diff_loc.view(t.uint8), world)
        all_gather_words(dist, r.view(t.uint8), r_loc.view(t.uint8), world)
        _capi.call("b2sr_pairwise_sum", dev.ptr(diff), n, dev.ptr(out), dev.stream())
        it += 1
        if float(out[0].item()) < epsilon:
            conv = True
            break
    return dev.to_host(r, np.float64, n), it, conv


def distributed_sssp(at: B2srMatrix, src: int, dist):
    """Unit-weight SSSP relaxation (algorithms.py:113-124) on ``at`` =
    transpose(drop_diagonal(a)), tile rows partitioned over ranks: per round
    the rank's rows of bff(at, dist, min-plus(1)) are relaxed into its slice,
    the slices are all-gathered and an all-reduce of the changed flags ends
    the loop exactly where the single-GPU driver stops.  Returns (dist, rounds)."""
    t = dev.torch()
    rank, world = dist.get_rank(), dist.get_world_size()
    n, d = at.n, at.dim
    b, e, v0, cnt, per = _slices(n, d, world, rank)
    blk = _new_handle("b2sr_row_block", at.handle().ptr, b, e, dev.stream())
    full = per * world
    dd = t.full((full,), float("inf"), dtype=t.float64, device=dev.device())
    dd[src] = 0.0
    y = t.zeros(per + 16, dtype=t.float64, device=dev.device())
    loc = t.zeros(per, dtype=t.float64, device=dev.device())
    flag = t.zeros(4, dtype=t.int32, device=dev.device())
    rounds = 0
    for _ in range(n - 1):
        _bff_block(blk, dd, 2, 1.0, y)  # B2SR_RING_MINPLUS, edge increment 1
        loc.copy_(dd[v0:v0 + per])
        flag.zero_()
        _capi.call("b2sr_min_relax", cnt, dev.ptr(loc), dev.ptr(y), dev.ptr(flag), dev.stream())
        all_gather_words(dist, dd.view(t.uint8), loc.view(t.uint8), world)
        dist.all_reduce(flag)
        rounds += 1
        if not int(flag[0].item()):
            break
    return dev.to_host(dd, np.float64, n), rounds


def distributed_triangle_count(lower: B2srMatrix, dist) -> int:
    """TC with the mask tile rows of L partitioned over ranks; L replicated."""
    rank, world = dist.get_rank(), dist.get_world_size()
    b, e = partition(lower.n_tile_rows, world, lower.dim)[rank]
    h = lower.handle()
    blk = _new_handle("b2sr_row_block", h.ptr, b, e, dev.stream())
    out = ctypes.c_int64()
    _capi.call("b2sr_bmm_sum_masked_bt", h.ptr, h.ptr, blk.ptr, ctypes.addressof(out), dev.stream())
    t = dev.torch()
    total = t.tensor([out.value], dtype=t.int64, device=dev.device())
    dist.all_reduce(total)
    return int(total.item())
