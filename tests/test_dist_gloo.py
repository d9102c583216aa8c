"""World-size-2 gloo tests (CPU) of the multi-GPU host logic in dist.py:
tile-row partitioning, the per-level frontier all-gather, the shared
termination test and the triangle-count all-reduce.  The per-rank compute
is the C oracle (test infrastructure) instead of the CUDA kernels; the loop,
buffers and exchange are the product's own code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as orc
from paper_2201_08560_b200 import dist as bdist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _block(m, b, e):
    n, d, trp, tci, tiles = m
    t0, t1 = int(trp[b]), int(trp[e])
    return (trp[b: e + 1] - trp[b]).astype(np.uint32), tci[t0:t1], tiles[t0:t1], b


class OracleBfsOps:
    """CPU stand-in for CudaBfsOps (same buffer layout: byte tensors of words)."""

    def __init__(self, block, n, d):
        self.trp, self.tci, self.tiles, self.row0 = block
        self.n, self.d = n, d
        self.wdt = orc.word_dtype(d)

    def buffers(self, global_bytes, block_bytes):
        z = lambda k: torch.zeros(k, dtype=torch.uint8)  # noqa: E731
        return z(global_bytes), z(global_bytes), z(block_bytes), torch.zeros(self.n, dtype=torch.float64), z(4)

    def _words(self, t):
        return t.numpy().view(self.wdt)

    def init(self, src, visited, frontier, levels):
        levels.fill_(np.inf)
        levels[src] = 0.0
        self._words(visited)[src // self.d] |= 1 << (src % self.d)
        self._words(frontier)[src // self.d] |= 1 << (src % self.d)

    def sweep(self, frontier, visited, nxt, sparse=False):
        fw, vw, out = self._words(frontier), self._words(visited), self._words(nxt)
        out[:] = 0
        ntr_global = orc.tile_rows(self.n, self.d)
        full = (1 << self.d) - 1
        for li in range(len(self.trp) - 1):
            g = self.row0 + li
            valid = full if (g + 1) * self.d <= self.n else (1 << (self.n - g * self.d)) - 1
            keep = ~int(vw[g]) & valid
            acc = 0
            for t in range(int(self.trp[li]), int(self.trp[li + 1])):
                xw = int(fw[self.tci[t]])
                for r in range(self.d):
                    if int(self.tiles[t, r]) & xw:
                        acc |= 1 << r
            out[li] = acc & keep
        assert ntr_global >= self.row0

    def update(self, frontier, visited, levels, level, anyflag):
        fw, vw = self._words(frontier), self._words(visited)
        lv = levels.numpy()
        found = False
        for i, w in enumerate(fw[: orc.tile_rows(self.n, self.d)]):
            w = int(w)
            if w:
                found = True
                vw[i] |= w
                for k in range(self.d):
                    if (w >> k) & 1:
                        lv[i * self.d + k] = level
        return found, int(sum(bin(int(w)).count("1") for w in fw[: orc.tile_rows(self.n, self.d)]))

    def levels_to_host(self, levels):
        return levels.numpy().copy()


def _worker(rank, world, port, scale, d, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 1 << scale
    rp, ci = orc.rmat_csr(scale, 8, seed=5)
    m = orc.csr_to_b2sr(n, rp, ci, d)
    at = orc.transpose(m)
    ntr = orc.tile_rows(n, d)
    b, e = bdist.partition(ntr, world, d)[rank]
    ops = OracleBfsOps(_block(at, b, e), n, d)
    runner = bdist.DistributedBfs(n, d, ntr, rank, world, ops, dist)
    deg = np.diff(rp.astype(np.int64))
    src = int(np.argmax(deg))
    levels, it = runner.run(src)
    # triangle count: mask rows partitioned, L replicated, one all-reduce
    lrp, lci = orc.lower_triangle(n, rp, ci)
    lo = orc.csr_to_b2sr(n, lrp, lci, d)
    mtrp = lo[2].copy()
    mtrp[: b + 1] = lo[2][b]
    mtrp[e:] = lo[2][e]
    mtrp = (mtrp - lo[2][b]).astype(np.uint32)
    t0, t1 = int(lo[2][b]), int(lo[2][e])
    mask = (n, d, mtrp, lo[3][t0:t1].copy(), lo[4][t0:t1].copy())
    part = orc.bmm_sum_masked(lo, orc.transpose(lo), mask)
    tot = torch.tensor([part], dtype=torch.int64)
    dist.all_reduce(tot)
    if rank == 0:
        q.put((levels, it, int(tot.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d", [4, 32])
def test_distributed_bfs_and_tc_world2(d):
    scale = 9
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, scale, d, q)) for r in range(2)]
    for p in procs:
        p.start()
    levels, it, tc = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    n = 1 << scale
    rp, ci = orc.rmat_csr(scale, 8, seed=5)
    m = orc.csr_to_b2sr(n, rp, ci, d)
    want, want_it = orc.bfs(m, int(np.argmax(np.diff(rp.astype(np.int64)))))
    assert levels.tobytes() == want.tobytes() and it == want_it
    assert tc == orc.triangle_count(n, rp, ci, d)


def test_partition_properties():
    for ntr in (1, 5, 33, 1000, 262144):
        for world in (1, 2, 4, 8):
            for d in (4, 8, 16, 32):
                parts = bdist.partition(ntr, world, d)
                assert parts[0][0] == 0 and parts[-1][1] == ntr
                assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
                wb = 4 if d == 32 else (2 if d == 16 else 1)
                assert (bdist.block_rows(ntr, world, d) * wb) % 4 == 0


def test_resolve_devices_and_row_cuts(monkeypatch):
    import numpy as np

    from paper_2201_08560_b200 import dist as bdist

    monkeypatch.delenv("B2SR_GPUS", raising=False)
    assert bdist.resolve_devices(None) == [None]
    assert bdist.resolve_devices(3) == [0, 1, 2]
    assert bdist.resolve_devices([1, 0]) == [1, 0]
    monkeypatch.setenv("B2SR_GPUS", "4")
    assert bdist.resolve_devices(None) == [0, 1, 2, 3]
    monkeypatch.setenv("B2SR_GPUS", "0,0")
    assert bdist.resolve_devices(None) == [0, 0]
    for bad in (0, [], [-1]):
        with pytest.raises(ValueError):
            bdist.resolve_devices(bad)
    rng = np.random.default_rng(0)
    lens = rng.integers(0, 50, 1000)
    trp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    for world, dim in ((2, 4), (3, 8), (8, 16), (5, 32)):
        cuts = bdist._row_cuts(trp, world, dim)
        align = 16 // (4 if dim == 32 else 2 if dim == 16 else 1)
        assert cuts[0] == 0 and cuts[-1] == 1000 and cuts == sorted(cuts) and len(cuts) == world + 1
        assert all(c % align == 0 or c == 1000 for c in cuts)
        tiles = [int(trp[cuts[r + 1]] - trp[cuts[r]]) for r in range(world)]
        assert max(tiles) - min(tiles) <= 2 * align * 50 + 1  # balanced up to the alignment granule
