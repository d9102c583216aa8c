"""GPU: the native row-partitioned drivers (b2sr_dist_*) against the oracle.

Only one GPU is available to this build, so the multi-rank level loop runs
as N thread-ranks sharing cuda:0 (b2sr_comm_init_local: every exchange is a
stream-ordered device copy behind host barriers, with NCCL's matching rules),
and the NCCL communicator itself runs as a world of one -- the same plan,
level loop and exchange calls the 8-GPU run makes.  Directed graphs make a
and at differ, so push (over a's blocks) and pull (over at's blocks) are
both checked; the shrunken hot cache forces the cold gathers at small n.
"""

import threading

import numpy as np
import pytest

import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import dist as bdist
from paper_2201_08560_b200 import rmat
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _run_ranks(world, fn):
    """fn(rank, comm, stream) on `world` threads, each with its own stream."""
    import torch

    comms = bdist.Comm.local(world)
    out, err = [None] * world, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                out[r] = fn(r, comms[r], st.cuda_stream)
                st.synchronize()
        except BaseException as e:  # noqa: BLE001 -- surfaced below
            err.append(e)

    ts = [threading.Thread(target=body, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=600)
    if err:
        raise err[0]
    return out


def _graph(scale, undirected, seed=5):
    csr = rmat.rmat_csr(scale, 16, seed=seed, undirected=undirected)
    return csr


@pytest.mark.parametrize("d", [4, 8])
@pytest.mark.parametrize("world", [1, 2, 3])
@pytest.mark.parametrize("undirected", [True, False])
def test_dist_bfs_thread_ranks(d, world, undirected, monkeypatch):
    monkeypatch.setenv("B2SR_HOT_BYTES", "2048")
    scale = 14
    csr = _graph(scale, undirected)
    n = csr.n
    m = b2.csr_to_b2sr(csr, d)
    at = b2.b2sr_transpose(m)
    ref = (n, d, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles)
    deg = np.diff(csr.row_ptr.astype(np.int64))
    srcs = [int(np.argmax(deg)), int(np.flatnonzero(deg > 0)[7])]
    want = [orc.bfs(ref, s) for s in srcs]

    def rank(r, comm, sp):
        plan = bdist.NativeDistributedBfs.from_matrices(comm, m, at)
        got = [plan.run(s, stream=sp) for s in srcs]
        return plan.rows, got

    res = _run_ranks(world, rank)
    rows = [r[0] for r in res]
    assert rows[0][0] == 0 and rows[-1][1] == m.n_tile_rows
    assert all(rows[i][1] == rows[i + 1][0] for i in range(world - 1))
    for r in range(world):
        for (lv, it), (wl, wit) in zip(res[r][1], want):
            assert lv.tobytes() == wl.tobytes() and it == wit


def test_dist_bfs_plan_from_host_blocks():
    """The e2e leg: every rank uploads only its rows of a and at from host
    arrays plus the global tile_row_ptr; same levels as the oracle."""
    d, world, scale = 4, 3, 13
    csr = _graph(scale, False, seed=9)
    n = csr.n
    m = b2.csr_to_b2sr(csr, d)
    at = b2.b2sr_transpose(m)
    ref = (n, d, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles)
    src = int(np.argmax(np.diff(csr.row_ptr.astype(np.int64))))
    want = orc.bfs(ref, src)
    ntr = m.n_tile_rows
    cuts = [0, (ntr // 3) // 16 * 16, (2 * ntr // 3) // 16 * 16, ntr]

    def host_block(mat, b, e):
        trp = mat.tile_row_ptr.astype(np.int64)
        t0, t1 = int(trp[b]), int(trp[e])
        return ((None, (trp[b:e + 1] - t0).astype(np.uint32)), (None, mat.tile_col_ind[t0:t1].copy()),
                (None, mat.bit_tiles[t0:t1].copy()))

    def rank(r, comm, sp):
        b, e = cuts[r], cuts[r + 1]
        ab = bdist.block_from_host(n, d, b, e, host_block(m, b, e))
        atb = bdist.block_from_host(n, d, b, e, host_block(at, b, e))
        plan = bdist.NativeDistributedBfs.from_blocks(comm, ab, atb, m.tile_row_ptr, at.tile_row_ptr)
        return plan.rows, plan.run(src, stream=sp)

    res = _run_ranks(world, rank)
    for r in range(world):
        assert res[r][0] == (cuts[r], cuts[r + 1])
        assert res[r][1][0].tobytes() == want[0].tobytes() and res[r][1][1] == want[1]


@pytest.mark.parametrize("d", [4, 8])
def test_dist_bfs_nccl_world_of_one(d):
    """The NCCL communicator (libnccl opened at run time) as a world of one."""
    csr = _graph(13, False, seed=3)
    m = b2.csr_to_b2sr(csr, d)
    at = b2.b2sr_transpose(m)
    src = int(np.argmax(np.diff(csr.row_ptr.astype(np.int64))))
    want = orc.bfs((csr.n, d, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles), src)
    comm = bdist.Comm.nccl_single()
    plan = bdist.NativeDistributedBfs.from_matrices(comm, m, at)
    lv, it = plan.run(src)
    assert lv.tobytes() == want[0].tobytes() and it == want[1]
    lower = b2.csr_to_b2sr(b2.algorithms._degree_oriented(_graph(13, True, seed=3)), d)
    cnt, cuts = bdist.native_triangle_count(comm, lower)
    assert cnt == b2.algorithms._tc_count(lower) and cuts == [0, lower.n_tile_rows]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("d", [4, 8])
def test_dist_tc_thread_ranks(world, d):
    scale = 13
    rp, ci = orc.rmat_csr(scale, 16, seed=4)
    n = 1 << scale
    want = orc.triangle_count(n, rp, ci, d)
    csr = b2.CsrMatrix(n, rp, ci)
    lower = b2.csr_to_b2sr(b2.algorithms._degree_oriented(csr), d)

    def rank(r, comm, sp):
        return bdist.native_triangle_count(comm, lower, stream=sp)

    res = _run_ranks(world, rank)
    for cnt, cuts in res:
        assert cnt == want
        assert cuts[0] == 0 and cuts[-1] == lower.n_tile_rows and cuts == sorted(cuts)


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
@pytest.mark.parametrize("d", [4, 8])
def test_bfs_devices_keyword(devices, d):
    """The drop-in bfs(a, src, devices=...) -- one process, one rank per listed
    device (repeated ordinals: thread-ranks on one GPU) -- equals the oracle,
    and a second call reuses the cached per-device plans."""
    csr = _graph(13, False, seed=11)
    m = b2.csr_to_b2sr(csr, d)
    ref = (csr.n, d, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles)
    deg = np.diff(csr.row_ptr.astype(np.int64))
    for src in (int(np.argmax(deg)), int(np.flatnonzero(deg > 0)[3])):
        lv, it = orc.bfs(ref, src)
        r = b2.bfs(m, src, devices=devices)
        assert r.per_vertex.tobytes() == lv.tobytes() and r.iterations == it
    assert len(m._dist) == 1
