"""Pin the C oracle (oracle/b2sr_oracle.c) to the reference's own outputs.

The golden vectors were produced by running the reference package unchanged
(tests/golden/make_golden.py).  Everything is compared bit-for-bit: integer
and bit outputs exactly, float64 outputs with ``tobytes()`` equality.
"""

import numpy as np
import pytest

from conftest import DIMS
from oracle import oracle as orc


def _csr(g, name):
    return g[f"{name}/row_ptr"], g[f"{name}/col_ind"]


def _cases(g):
    return [c for c in g.cases]


def test_conversion_and_transpose(golden):
    for c in _cases(golden):
        name, n = c["name"], c["n"]
        rp, ci = _csr(golden, name)
        for d in DIMS:
            m = orc.csr_to_b2sr(n, rp, ci, d)
            ref = golden.matrix(name, d)
            for got, want in zip(m[2:], ref[2:]):
                assert got.dtype == want.dtype and np.array_equal(got, want), (name, d)
            t = orc.transpose(m)
            reft = golden.matrix(name, d, transposed=True)
            for got, want in zip(t[2:], reft[2:]):
                assert np.array_equal(got, want), (name, d)
            rp2, ci2 = orc.b2sr_to_csr(m)
            assert np.array_equal(rp2, rp) and np.array_equal(ci2, ci)
            assert np.array_equal(orc.used_columns(m), golden[f"{name}/d{d}/used"])


def test_bmv_kernels(golden):
    for c in _cases(golden):
        name, n = c["name"], c["n"]
        g = lambda k: golden[f"{name}/{k}"]  # noqa: E731
        for d in DIMS:
            m = golden.matrix(name, d)
            p = lambda k: golden[f"{name}/d{d}/{k}"]  # noqa: E731
            xw = orc.pack_bits(g("xb"), d)
            kw = orc.pack_bits(g("keep"), d)
            assert np.array_equal(orc.bmv_bbb(m, xw), p("bbb"))
            assert np.array_equal(orc.bmv_bbb(m, xw, kw), p("bbb_m"))
            assert orc.bmv_bbf(m, xw).tobytes() == p("bbf").tobytes()
            assert orc.bmv_bbf(m, xw, kw).tobytes() == p("bbf_m").tobytes()
            assert orc.bmv_bff(m, g("xf"), "arithmetic").tobytes() == p("bff_ar").tobytes()
            assert orc.bmv_bff(m, g("xf"), "arithmetic", keep_words=kw).tobytes() == p("bff_ar_m").tobytes()
            assert orc.bmv_bff(m, g("xm"), "minplus", 1.0).tobytes() == p("bff_mp1").tobytes()
            assert orc.bmv_bff(m, g("xm"), "minplus", 1.0, keep_words=kw).tobytes() == p("bff_mp1_m").tobytes()
            assert orc.bmv_bff(m, g("xm"), "minplus", 0.0).tobytes() == p("bff_mp0").tobytes()
            assert orc.bmv_bff(m, g("xp"), "maxtimes").tobytes() == p("bff_mx").tobytes()
            if n:
                got = orc.bmv_bff(m, g("xp"), "arithmetic", scale=p("scale"))
                assert got.tobytes() == p("bff_sc").tobytes()


def test_bmm(golden):
    for c in _cases(golden):
        name, n = c["name"], c["n"]
        for d in DIMS:
            a = golden.matrix(name, d)
            b = orc.csr_to_b2sr(n, golden[f"{name}/b_row_ptr"], golden[f"{name}/b_col_ind"], d)
            m = orc.csr_to_b2sr(n, golden[f"{name}/m_row_ptr"], golden[f"{name}/m_col_ind"], d)
            assert orc.bmm_sum(a, b) == int(golden[f"{name}/d{d}/bmm"][0])
            if f"{name}/d{d}/bmm_m" in golden:
                assert orc.bmm_sum_masked(a, b, m) == int(golden[f"{name}/d{d}/bmm_m"][0])
                assert orc.bmm_sum_masked(a, a, a) == int(golden[f"{name}/d{d}/bmm_aa"][0])


def test_algorithms(golden):
    for c in _cases(golden):
        name, n = c["name"], c["n"]
        src = int(golden[f"{name}/src"][0])
        deg = golden[f"{name}/deg"]
        for d in DIMS:
            p = lambda k: golden[f"{name}/d{d}/{k}"]  # noqa: E731
            m = golden.matrix(name, d)
            lv, it = orc.bfs(m, src)
            assert lv.tobytes() == p("bfs").tobytes() and it == p("bfs_it")[0]
            ds, it = orc.sssp(m, src)
            assert ds.tobytes() == p("sssp").tobytes() and it == p("sssp_it")[0]
            rank, it, conv = orc.pagerank(golden.matrix(name, d, transposed=True), deg)
            assert rank.tobytes() == p("pr").tobytes()
            assert [it, int(conv)] == p("pr_it").tolist()
            if c["symmetric"]:
                lab, it = orc.connected_components(m)
                assert lab.tobytes() == p("cc").tobytes() and it == p("cc_it")[0]
                if f"{name}/d{d}/tc" in golden:
                    rp, ci = _csr(golden, name)
                    assert orc.triangle_count(n, rp, ci, d) == int(p("tc")[0])


def test_pairwise_matches_numpy():
    rng = np.random.default_rng(7)
    for n in (0, 1, 7, 8, 9, 127, 128, 129, 1000, 65537):
        a = rng.random(n) * 10.0 ** rng.integers(-8, 8, n)
        assert orc.pairwise_sum(a) == a.sum()


def test_bff_errors(golden):
    m = golden.matrix("rnd8", 8)
    n = m[0]
    with pytest.raises(orc.OracleError):
        orc.bmv_bff(m, np.zeros(n), "boolean")
    with pytest.raises(orc.OracleError):
        orc.bmv_bff(m, np.zeros(n), "minplus", 1.0, scale=np.ones(n))
    used = orc.used_columns(m)
    sc = np.ones(n)
    sc[np.flatnonzero(used)[0]] = 0.0
    with pytest.raises(orc.OracleError):
        orc.bmv_bff(m, np.zeros(n), "arithmetic", scale=sc)
