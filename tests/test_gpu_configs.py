"""GPU parity at the full sizes of BASELINE.json configs[0..3].

Each test builds the graph twice -- the device generator + device COO->CSR
+ device conversion (the product path), and the CPU twin + the C oracle's
own csr_to_b2sr (oracle/, the restated reference) -- so conversion is
checked at full size too, then compares every output the config names:

  configs[0]  s16, B2SR-32: csr_to_b2sr + bbb / bbf / bff (+ masked), the
              reference bench's vectors (cli.py:236-240)
  configs[1]  s22 BFS at d = 4 / 8 / 16 / 32 (levels + sweep count) and the
              masked K4 sweep behind the roofline figure
  configs[2]  s20 triangle count at d = 4, 8 against the reference's own
              ID-ordered lower-triangle SpGEMM (algorithms.py:199-215)
  configs[3]  s24 PageRank / SSSP / CC, oracle converting from CSR itself

Bar: bit-exact (``tobytes()`` for float64) everywhere; PageRank additionally
reports the north-star tolerance (relative L1 <= 1e-5) it sits inside.
"""

import numpy as np
import pytest

import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat
from conftest import bfs_all_paths
from oracle import oracle as orc

pytestmark = pytest.mark.gpu


def _graph(scale, undirected=True):
    """(device CsrMatrix, oracle (row_ptr, col_ind)) of the same R-MAT graph;
    the two generators are twins, checked here at full size."""
    csr = rmat.rmat_csr(scale, 16, seed=1, undirected=undirected)
    rp, ci = orc.rmat_csr(scale, 16, seed=1, undirected=undirected)
    assert np.array_equal(csr.row_ptr, rp) and np.array_equal(csr.col_ind, ci)
    return csr, (rp, ci)


def _same_layout(m, ref):
    assert m.tile_row_ptr.dtype == ref[2].dtype and np.array_equal(m.tile_row_ptr, ref[2])
    assert np.array_equal(m.tile_col_ind, ref[3])
    assert m.bit_tiles.dtype == ref[4].dtype and np.array_equal(m.bit_tiles, ref[4])


def _roots(rp, k, seed):
    deg = np.diff(rp.astype(np.int64))
    rng = np.random.default_rng(seed)
    return [int(v) for v in rng.choice(np.flatnonzero(deg > 0), size=k, replace=False)]


@pytest.mark.parametrize("undirected", [False, True])
def test_config0_s16_d32_conversion_and_bmv(undirected):
    scale, d = 16, 32
    n = 1 << scale
    csr, (rp, ci) = _graph(scale, undirected)
    m = b2.csr_to_b2sr(csr, d)
    ref = orc.csr_to_b2sr(n, rp, ci, d)
    _same_layout(m, ref)
    rng = np.random.default_rng(1)  # the reference bench's vectors (cli.py:236-240)
    xb = rng.random(n) < 0.5
    xf = rng.random(n)
    keep = np.random.default_rng(2).random(n) < 0.5
    xw, kw = orc.pack_bits(xb, d), orc.pack_bits(keep, d)
    X, K = b2.BitVector.from_bools(xb, d), b2.BitVector.from_bools(keep, d)
    assert np.array_equal(b2.bmv_bin_bin_bin(m, X).words, orc.bmv_bbb(ref, xw))
    assert np.array_equal(b2.bmv_bin_bin_bin_masked(m, X, K).words, orc.bmv_bbb(ref, xw, kw))
    assert b2.bmv_bin_bin_full(m, X).tobytes() == orc.bmv_bbf(ref, xw).tobytes()
    assert b2.bmv_bin_bin_full_masked(m, X, K).tobytes() == orc.bmv_bbf(ref, xw, kw).tobytes()
    assert b2.bmv_bin_full_full(m, xf, b2.ARITHMETIC).tobytes() == orc.bmv_bff(ref, xf, "arithmetic").tobytes()
    got = b2.bmv_bin_full_full_masked(m, xf, b2.ARITHMETIC, K)
    assert got.tobytes() == orc.bmv_bff(ref, xf, "arithmetic", keep_words=kw).tobytes()
    assert (b2.bmv_bin_full_full(m, xf, b2.min_plus(1)).tobytes()
            == orc.bmv_bff(ref, xf, "minplus", 1.0).tobytes())
    t = b2.b2sr_transpose(m)
    _same_layout(t, orc.transpose(ref))


@pytest.fixture(scope="module")
def s22():
    return _graph(22)


@pytest.mark.parametrize("d", [4, 8, 16, 32])
def test_config1_s22_bfs(s22, d):
    """BFS levels and sweep counts from two bench-style roots at every tile
    width of the sweep; conversion checked against the oracle's own."""
    import torch

    csr, (rp, ci) = s22
    n = csr.n
    m = b2.csr_to_b2sr(csr, d)
    ref = orc.csr_to_b2sr(n, rp, ci, d)
    _same_layout(m, ref)
    if d == 4:  # the roofline kernel: masked full sweep, 50 % random x and keep
        rng = np.random.default_rng(11)
        xb, keep = rng.random(n) < 0.5, rng.random(n) < 0.5
        got = b2.bmv_bin_bin_bin_masked(m, b2.BitVector.from_bools(xb, d), b2.BitVector.from_bools(keep, d))
        assert np.array_equal(got.words, orc.bmv_bbb(ref, orc.pack_bits(xb, d), orc.pack_bits(keep, d)))
    for src in _roots(rp, 2, 8):
        # d >= 16: the oracle takes the (undirected, hence symmetric) matrix as
        # its own transpose -- its transpose costs 15-30 s there; d <= 8 transposes
        lv, it = orc.bfs(ref, src, symmetric=d >= 16)
        r = bfs_all_paths(b2, m, src) if d <= 8 else b2.bfs(m, src)
        assert r.per_vertex.tobytes() == lv.tobytes() and r.iterations == it, (d, src)
    del m, ref
    torch.cuda.empty_cache()


@pytest.mark.parametrize("d", [4, 8])
def test_config2_s20_triangle_count(d):
    """The device count (degree-oriented DAG, K8) against the reference
    algorithm on the ID-ordered strict lower triangle, run by the oracle."""
    csr, (rp, ci) = _graph(20)
    got = b2.triangle_count(csr, d)
    assert got.count == orc.triangle_count(csr.n, rp, ci, d)
    assert got.per_vertex is None and got.iterations == 1


def test_config3_s24_pagerank_sssp_cc():
    import torch

    scale, d = 24, 4
    csr, (rp, ci) = _graph(scale)
    n = csr.n
    m = b2.csr_to_b2sr(csr, d)
    ref = orc.csr_to_b2sr(n, rp, ci, d)
    _same_layout(m, ref)
    at = b2.b2sr_transpose(m)
    ref_t = orc.transpose(ref)
    _same_layout(at, ref_t)
    deg = np.diff(rp.astype(np.int64)).astype(np.float64)
    # PageRank on the transposed adjacency (algorithms.py:127-163)
    pr = b2.pagerank(at, deg)
    want, it, conv = orc.pagerank(ref_t, deg)
    rel_l1 = np.abs(pr.per_vertex - want).sum() / np.abs(want).sum()
    assert rel_l1 <= 1e-5 and pr.iterations == it and pr.converged == conv
    assert pr.per_vertex.tobytes() == want.tobytes()  # the default driver is bit-exact
    # the documented fast mode (float32 x, order-free float64 sums) sits inside the tolerance
    import os

    os.environ["B2SR_PR_MODE"] = "fast"
    try:
        prf = b2.pagerank(at, deg)
    finally:
        del os.environ["B2SR_PR_MODE"]
    rel_f = np.abs(prf.per_vertex - want).sum() / np.abs(want).sum()
    assert rel_f <= 1e-5 and prf.iterations == it and prf.converged == conv, rel_f
    # SSSP: the graph is loop-free, so drop_diagonal(m) = m and its transpose is ref_t
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp.astype(np.int64)))
    assert not np.any(rows == ci)
    del rows
    src = int(np.argmax(deg))
    ss = b2.sssp(m, src)
    dist, sit = orc.sssp(ref, src, at=ref_t)
    assert ss.per_vertex.tobytes() == dist.tobytes() and ss.iterations == sit
    # CC (symmetric input)
    cc = b2.connected_components(m)
    lab, _ = orc.connected_components(ref)
    assert cc.per_vertex.tobytes() == lab.tobytes()
    del m, at
    torch.cuda.empty_cache()
