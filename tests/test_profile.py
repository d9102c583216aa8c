"""Tile-width sampler (profile.py) against the reference's own reports.

tests/golden/golden_profile.json holds b2sr.sample_profile(...).to_report()
of the reference for the golden graphs and R-MAT s12/s14 at several sample
counts and seeds (tests/golden/make_golden_profile.py).  The GPU sampler
draws the same sample with the same generator calls and counts tiles on the
device; its report must equal the reference's exactly (floats included).
"""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2201_08560_b200 as b2
from oracle import oracle as orc

HERE = Path(__file__).resolve().parent


@pytest.fixture(scope="module")
def reports():
    return json.loads((HERE / "golden" / "golden_profile.json").read_text())


def _graph(golden, name):
    if name.startswith("rmat") and name[4:].isdigit() and int(name[4:]) >= 12:
        rp, ci = orc.rmat_csr(int(name[4:]), 16, seed=1)
        return b2.CsrMatrix(len(rp) - 1, rp, ci)
    rp, ci = golden[f"{name}/row_ptr"], golden[f"{name}/col_ind"]
    return b2.CsrMatrix(len(rp) - 1, rp, ci)


def test_argument_checks():
    """Validation happens before any device work (profile.py:81-87)."""
    csr = b2.CsrMatrix(10, np.zeros(11, np.uint32), np.zeros(0, np.uint32))
    for bad in (0, 4, -1):  # ceil(10/4) = 3 tile rows at width 4
        with pytest.raises(ValueError):
            b2.sample_profile(csr, bad, 0)


def test_report_fixture_is_complete(reports):
    kinds = {(r["graph"], r["sample_count"], r["seed"]) for r in reports}
    assert len(kinds) == len(reports) >= 100
    for r in reports:
        rep = r["report"]
        assert rep["kind"] == "profile" and set(rep["tileDims"]) == {"4", "8", "16", "32"}


@pytest.mark.gpu
def test_sample_profile_matches_reference(golden, reports):
    cache = {}
    for r in reports:
        name = r["graph"]
        if name not in cache:
            cache[name] = _graph(golden, name)
        got = b2.sample_profile(cache[name], r["sample_count"], r["seed"]).to_report()
        assert json.loads(json.dumps(got)) == r["report"], (name, r["sample_count"], r["seed"])
