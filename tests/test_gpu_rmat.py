"""GPU: the device R-MAT generator and COO->CSR equal their CPU twins, and
full-size (BASELINE configs) properties hold where the oracle is too slow."""

import numpy as np
import pytest

import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat
from conftest import bfs_all_paths
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [4, 10, 16])
def test_rmat_matches_cpu_twin(scale):
    src, dst = rmat.rmat_edges(scale, 16, seed=1)
    s_ref, d_ref = orc.rmat_edges(scale, 16, seed=1)
    assert np.array_equal(src.cpu().numpy().astype(np.uint32), s_ref)
    assert np.array_equal(dst.cpu().numpy().astype(np.uint32), d_ref)
    for undirected in (True, False):
        csr = rmat.rmat_csr(scale, 16, seed=1, undirected=undirected)
        rp, ci = orc.rmat_csr(scale, 16, seed=1, undirected=undirected)
        assert np.array_equal(csr.row_ptr, rp) and np.array_equal(csr.col_ind, ci)


def test_from_coo_device_matches_host():
    t = __import__("torch")
    rng = np.random.default_rng(3)
    n = 1000
    r = rng.integers(0, n, 20000)
    c = rng.integers(0, n, 20000)
    host = b2.CsrMatrix.from_coo(n, r, c)
    devm = b2.CsrMatrix.from_coo(n, t.tensor(r, device="cuda"), t.tensor(c, device="cuda"))
    assert devm == host


def test_scale20_properties():
    """s20 (BASELINE config 3 size): layout invariants and identities at full size."""
    csr = rmat.rmat_csr(20, 16, seed=1)
    n = csr.n
    for d in (4, 32):
        m = b2.csr_to_b2sr(csr, d)
        assert m.nnz == csr.nnz
        # symmetric input: transpose is the identity, and an involution
        t = b2.b2sr_transpose(m)
        assert t == m
        assert b2.b2sr_to_csr(m) == csr
        # bbf with x = all ones equals the out-degree; bbb with all ones = deg > 0
        ones = b2.BitVector.from_bools(np.ones(n, bool), d)
        deg = np.diff(csr.row_ptr.astype(np.int64))
        assert np.array_equal(b2.bmv_bin_bin_full(m, ones), deg.astype(np.float64))
        assert np.array_equal(b2.bmv_bin_bin_bin(m, ones).to_bools(), deg > 0)
        # bmm_sum(A, A) = sum_k deg(k)^2 for symmetric A
        assert b2.bmm_bin_bin_sum(m, m) == int((deg * deg).sum()) if n ** 3 < 2 ** 63 else True
        # BFS levels: |level(u) - level(v)| <= 1 on every edge; src level 0
        src = int(np.argmax(deg))
        lv = bfs_all_paths(b2, m, src).per_vertex
        rows = np.repeat(np.arange(n), deg)
        cols = csr.col_ind.astype(np.int64)
        a, bb = lv[rows], lv[cols]
        fin = np.isfinite(a) | np.isfinite(bb)
        assert np.all(np.isfinite(a[fin]) & np.isfinite(bb[fin]))
        assert np.abs(a[fin] - bb[fin]).max() <= 1 and lv[src] == 0


@pytest.mark.parametrize("d", [4, 8, 32])
def test_scale21_against_oracle(d):
    """n = 2^21: more tile columns than the shared-memory hot cache holds at
    d = 4, 8 (hot and cold x gathers in the flat stream), masked bbb and BFS
    against the C oracle."""
    scale = 21
    n = 1 << scale
    csr = rmat.rmat_csr(scale, 8, seed=2)
    rp, ci = csr.row_ptr, csr.col_ind
    m = b2.csr_to_b2sr(csr, d)
    ref = (n, d, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles)
    rng = np.random.default_rng(21)
    xb = rng.random(n) < 0.5
    keep = rng.random(n) < 0.5
    xw, kw = orc.pack_bits(xb, d), orc.pack_bits(keep, d)
    got = b2.bmv_bin_bin_bin_masked(m, b2.BitVector.from_bools(xb, d), b2.BitVector.from_bools(keep, d))
    assert np.array_equal(got.words, orc.bmv_bbb(ref, xw, kw))
    src = int(np.argmax(np.diff(rp.astype(np.int64))))
    lv, it = orc.bfs(ref, src)
    r = bfs_all_paths(b2, m, src)
    assert r.per_vertex.tobytes() == lv.tobytes() and r.iterations == it


def _dist_bfs_worker(rank, world, port, scale, d, src, q):
    import os

    import torch
    import torch.distributed as tdist

    from paper_2201_08560_b200 import dist as bdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    csr = rmat.rmat_csr(scale, 16, seed=5)
    at = b2.b2sr_transpose(b2.csr_to_b2sr(csr, d))
    lv, it = bdist.DistributedBfs.from_matrix(at, tdist).run(src)
    # the e2e leg: a rank's block re-uploaded from host arrays gives the same levels
    b, e = bdist.partition(at.n_tile_rows, world, d)[rank]
    blk = b2.formats._new_handle("b2sr_row_block", at.handle().ptr, b, e, 0)
    hb = bdist.block_from_host(csr.n, d, b, e, bdist.block_to_host(blk))
    lv2, it2 = bdist.DistributedBfs.from_block(hb, csr.n, d, tdist).run(src)
    if rank == 0:
        q.put((lv.tobytes(), it, lv2.tobytes(), it2))
    tdist.destroy_process_group()


@pytest.mark.parametrize("d", [4, 8, 32])
def test_row_partitioned_bfs_two_ranks_one_gpu(d):
    """dist.py with the real kernels: 2 ranks (gloo, sharing cuda:0) give the
    oracle's levels and sweep count, also from blocks uploaded from host."""
    import socket

    import torch.multiprocessing as mp

    scale = 14
    rp, ci = orc.rmat_csr(scale, 16, seed=5)
    n = 1 << scale
    src = int(np.argmax(np.diff(rp.astype(np.int64))))
    lv_ref, it_ref = orc.bfs(orc.csr_to_b2sr(n, rp, ci, d), src)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dist_bfs_worker, args=(r, 2, port, scale, d, src, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=300)
    for p in ps:
        p.join(timeout=60)
    assert got[0] == lv_ref.tobytes() and got[1] == it_ref
    assert got[2] == lv_ref.tobytes() and got[3] == it_ref


def _dist_float_worker(rank, world, port, scale, d, src, q):
    import os

    import torch
    import torch.distributed as tdist

    from paper_2201_08560_b200 import dist as bdist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    csr = rmat.rmat_csr(scale, 16, seed=7)
    m = b2.csr_to_b2sr(csr, d)
    deg = np.diff(csr.row_ptr.astype(np.int64)).astype(np.float64)
    pr, pit, pconv = bdist.distributed_pagerank(b2.b2sr_transpose(m), deg, tdist)
    ss, sit = bdist.distributed_sssp(b2.b2sr_transpose(b2.formats.drop_diagonal(m)), src, tdist)
    if rank == 0:
        q.put((pr.tobytes(), pit, pconv, ss.tobytes(), sit))
    tdist.destroy_process_group()


@pytest.mark.parametrize("d", [4, 8])
def test_row_partitioned_pagerank_sssp_two_ranks_one_gpu(d, monkeypatch):
    """dist.py float-gather drivers with the real kernels (2 ranks sharing
    cuda:0 over gloo, small segmented-plan threshold so both gather paths run):
    PageRank and SSSP give the single-GPU drivers' bits and iteration counts."""
    import socket

    import torch.multiprocessing as mp

    monkeypatch.setenv("B2SR_VLONG_TILES", "24")
    scale = 13
    csr = rmat.rmat_csr(scale, 16, seed=7)
    m = b2.csr_to_b2sr(csr, d)
    deg = np.diff(csr.row_ptr.astype(np.int64)).astype(np.float64)
    src = int(np.argmax(deg))
    want_pr = b2.pagerank(b2.b2sr_transpose(m), deg)
    want_ss = b2.sssp(m, src)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_dist_float_worker, args=(r, 2, port, scale, d, src, q)) for r in range(2)]
    for p in ps:
        p.start()
    got = q.get(timeout=120)
    for p in ps:
        p.join(timeout=60)
    assert got[0] == want_pr.per_vertex.tobytes() and got[1] == want_pr.iterations and got[2] == want_pr.converged
    assert got[3] == want_ss.per_vertex.tobytes() and got[4] == want_ss.iterations


@pytest.mark.parametrize("pack", ["tiles", "all", "split"])
def test_large_host_upload_paths(tmp_path, monkeypatch, pack):
    """Host-array uploads above the staging threshold (staging.cu): the
    staged copy of tile_col_ind and the nibble-packed d=4 tile upload give the
    device the caller's exact bytes; a d=4 tile with a high nibble set still
    reaches the device check and raises the reference constructor's message."""
    from paper_2201_08560_b200.errors import FormatError

    monkeypatch.setenv("B2SR_H2D_PACK", pack)
    csr = rmat.rmat_csr(18, 16, seed=4)  # ~7.7 M tiles at d=4: 31 MB of tiles, past the 16 MB threshold
    for d in (4, 8):
        m = b2.csr_to_b2sr(csr, d)
        trp, tci, tiles = m.tile_row_ptr.copy(), m.tile_col_ind.copy(), m.bit_tiles.copy()
        h = b2.B2srMatrix(csr.n, d, trp, tci, tiles)  # host-built: uploaded on first use
        assert h == m
        p = tmp_path / f"m{d}.b2sr"
        b2.save_b2sr(m, p)
        back = b2.load_b2sr(p)  # straight to HBM through the device check
        assert back == m
        assert back.bit_tiles.tobytes() == tiles.tobytes() and back.tile_col_ind.tobytes() == tci.tobytes()
    m = b2.csr_to_b2sr(csr, 4)
    trp, tci, tiles = m.tile_row_ptr.copy(), m.tile_col_ind.copy(), m.bit_tiles.copy()
    tiles[len(tiles) // 2] |= 0x10  # a high nibble in a row byte of a 4x4 tile
    raw = (b2.formats._HEADER.pack(b2.formats._MAGIC, b2.formats._VERSION, csr.n, 4, len(trp) - 1, len(tci))
           + trp.astype("<u4").tobytes() + tci.astype("<u4").tobytes() + tiles.astype(np.uint8).tobytes())
    q = tmp_path / "bad.b2sr"
    q.write_bytes(raw)
    with pytest.raises(FormatError) as e_dev:
        b2.load_b2sr(q)
    with pytest.raises(FormatError) as e_host:
        b2.B2srMatrix(csr.n, 4, trp, tci, tiles)
    assert str(e_dev.value) == str(e_host.value)
    # a tile column past the packed width (>= 2^ceil(log2 ntr)): the bit-packed
    # column upload falls back to the plain copy, the device check reports it
    trp, tci, tiles = m.tile_row_ptr.copy(), m.tile_col_ind.copy(), m.bit_tiles.copy()
    tci[len(tci) // 3] = 0xFFFFFFF0
    raw = (b2.formats._HEADER.pack(b2.formats._MAGIC, b2.formats._VERSION, csr.n, 4, len(trp) - 1, len(tci))
           + trp.astype("<u4").tobytes() + tci.astype("<u4").tobytes() + tiles.astype(np.uint8).tobytes())
    q.write_bytes(raw)
    with pytest.raises(FormatError) as e_dev:
        b2.load_b2sr(q)
    with pytest.raises(FormatError) as e_host:
        b2.B2srMatrix(csr.n, 4, trp, tci, tiles)
    assert str(e_dev.value) == str(e_host.value)


@pytest.mark.parametrize("logn", [20, 25])
def test_host_upload_split_columns(tmp_path, logn):
    """The default host upload splits tile_col_ind into a u16 stream plus the
    column bits above 16 (staging.cu SPLIT): a nibble per column when the
    columns need <= 20 bits (2^20 vertices at d=4: 18 bits), a byte up to 24
    (2^25 vertices: 23 bits).  The device gets the caller's exact bytes, and a
    column past the packed width falls back to the plain copy and raises the
    reference constructor's message."""
    from paper_2201_08560_b200.errors import FormatError

    n = 1 << logn
    rng = np.random.default_rng(logn)
    key = np.unique(rng.integers(0, n, 4_500_000, dtype=np.int64) * n + rng.integers(0, n, 4_500_000, dtype=np.int64))
    rows, cols = (key // n).astype(np.uint32), (key % n).astype(np.uint32)
    row_ptr = np.zeros(n + 1, dtype=np.uint32)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    csr = b2.CsrMatrix(n, row_ptr, cols)
    m = b2.csr_to_b2sr(csr, 4)
    assert m.num_tiles * 8 > (16 << 20)  # past the staging threshold
    trp, tci, tiles = m.tile_row_ptr.copy(), m.tile_col_ind.copy(), m.bit_tiles.copy()
    h = b2.B2srMatrix(n, 4, trp, tci, tiles)
    assert h == m
    hb = b2.formats.B2srMatrix._wrap(b2.formats._new_handle("b2sr_transpose", h.handle().ptr, 0))
    assert hb == b2.b2sr_transpose(m)
    bad = tci.copy()
    bad[len(bad) // 2] = np.uint32(n)  # >= ntr, and past 2^ceil(log2 ntr)
    raw = (b2.formats._HEADER.pack(b2.formats._MAGIC, b2.formats._VERSION, n, 4, len(trp) - 1, len(bad))
           + trp.astype("<u4").tobytes() + bad.astype("<u4").tobytes() + tiles.astype(np.uint8).tobytes())
    q = tmp_path / "bad.b2sr"
    q.write_bytes(raw)
    with pytest.raises(FormatError) as e_dev:
        b2.load_b2sr(q)  # read straight into the staged upload, checked on the device
    with pytest.raises(FormatError) as e_host:
        b2.B2srMatrix(n, 4, trp, bad, tiles)
    assert str(e_dev.value) == str(e_host.value)
