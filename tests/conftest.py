"""Shared test setup: the ``gpu`` marker, repo on sys.path, golden fixtures."""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
DIMS = (4, 8, 16, 32)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


class Golden:
    """Lazy view over tests/golden/golden.npz (written by make_golden.py)."""

    def __init__(self):
        self._z = np.load(GOLDEN / "golden.npz")
        self.cases = json.loads((GOLDEN / "manifest.json").read_text())["cases"]

    def __getitem__(self, key):
        return self._z[key]

    def __contains__(self, key):
        return key in self._z.files

    def matrix(self, name, d, transposed=False):
        c = next(c for c in self.cases if c["name"] == name)
        p = f"{name}/d{d}/" + ("t_" if transposed else "")
        return (c["n"], d, self[p + "trp"], self[p + "tci"], self[p + "tiles"])


@pytest.fixture(scope="session")
def golden():
    return Golden()


def random_pattern(rng, n, density, symmetric=False):
    """(row_ptr, col_ind) of an i.i.d. random n x n pattern."""
    mask = rng.random((n, n)) < density
    if symmetric:
        mask |= mask.T
        np.fill_diagonal(mask, False)
    r, c = np.nonzero(mask)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    return np.cumsum(rp).astype(np.uint32), c.astype(np.uint32)


def bfs_all_paths(b2, m, src):
    """bfs() through both device paths: push-only levels on a matrix without a
    transpose (d = 4, 8), then the direction-optimizing push/pull driver once
    the transpose is cached.  Both must agree bit for bit; returns the latter."""
    first = b2.bfs(m, src)
    b2.b2sr_transpose(m)  # cached on m: the next call takes the transposed path
    second = b2.bfs(m, src)
    assert first.per_vertex.tobytes() == second.per_vertex.tobytes()
    assert first.iterations == second.iterations
    return second
