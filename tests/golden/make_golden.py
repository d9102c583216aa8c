"""Generate the golden fixtures by running the REFERENCE package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``b2sr`` 0.1.0 unchanged from /root/reference/pkg/src and records
its outputs for seeded inputs into ``tests/golden/golden.npz`` (+ a JSON
manifest).  The fixtures travel with the repo; /root/reference does not, so
GPU parity tests compare against these files and against the C oracle.

Inputs:
  * ``rnd*``  -- i.i.d. random directed patterns, n in [1, 200] (the
    reference's own conftest style, pkg/tests/conftest.py:7-11),
  * ``sym*``  -- random symmetric loop-free patterns (conftest.py:14-21),
  * ``rmat*`` -- R-MAT graphs from this repo's counter-based generator
    (oracle.rmat_csr, the CPU twin of csrc/rmat.cu),
  * ``empty`` -- an n=6 matrix without entries (test_kernels.py:168-177).
"""

from __future__ import annotations

import json
import sys
import zlib
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(ROOT))

import b2sr  # noqa: E402  (the reference, not this repo)
from b2sr import (  # noqa: E402
    ARITHMETIC, MAX_TIMES, AlgoParams, BitVector, CsrMatrix, b2sr_transpose, bfs, bmm_bin_bin_sum,
    bmm_bin_bin_sum_masked, bmv_bin_bin_bin, bmv_bin_bin_bin_masked, bmv_bin_bin_full,
    bmv_bin_bin_full_masked, bmv_bin_full_full, bmv_bin_full_full_masked, connected_components,
    csr_to_b2sr, min_plus, pagerank, sssp, triangle_count,
)
from b2sr.kernels import used_columns  # noqa: E402

assert "reference" in b2sr.__file__, b2sr.__file__

from oracle import oracle  # noqa: E402

DIMS = (4, 8, 16, 32)


def rand_pattern(rng, n, density, symmetric=False):
    mask = rng.random((n, n)) < density
    if symmetric:
        mask |= mask.T
        np.fill_diagonal(mask, False)
    r, c = np.nonzero(mask)
    return CsrMatrix.from_coo(n, r, c)


def main():
    out: dict[str, np.ndarray] = {}
    manifest = {"cases": []}
    rng = np.random.default_rng(20260417)

    cases = []
    for i, n in enumerate([1, 2, 5, 17, 31, 33, 64, 65, 100, 129, 150, 200]):
        dens = float(np.exp(rng.uniform(np.log(0.005), np.log(0.3))))
        cases.append((f"rnd{i}", rand_pattern(rng, n, dens), False))
    cases.append(("empty", CsrMatrix(6, [0] * 7, []), False))
    for i, n in enumerate([3, 9, 40, 77, 120, 200]):
        dens = float(np.exp(rng.uniform(np.log(0.01), np.log(0.2))))
        cases.append((f"sym{i}", rand_pattern(rng, n, dens, symmetric=True), True))
    for scale in (8, 10):
        rp, ci = oracle.rmat_csr(scale, 16, seed=1, undirected=True)
        cases.append((f"rmat{scale}", CsrMatrix(1 << scale, rp, ci), True))
    rp, ci = oracle.rmat_csr(9, 8, seed=3, undirected=False)
    cases.append(("rmat9dir", CsrMatrix(1 << 9, rp, ci), False))

    for name, csr, symmetric in cases:
        n = csr.n
        crng = np.random.default_rng(zlib.crc32(name.encode()))
        out[f"{name}/row_ptr"] = csr.row_ptr
        out[f"{name}/col_ind"] = csr.col_ind
        xb = crng.random(n) < 0.5
        keep = crng.random(n) < 0.5
        xf = crng.standard_normal(n) * crng.uniform(0.1, 100)
        xm = np.where(crng.random(n) < 0.3, np.inf, crng.integers(0, 50, n).astype(np.float64))
        xp = crng.random(n)
        deg = np.diff(csr.row_ptr.astype(np.int64)).astype(np.float64)
        src = int(crng.integers(0, n))
        bcsr = rand_pattern(crng, n, 0.1)
        mcsr = rand_pattern(crng, n, 0.1)
        for k, v in dict(xb=xb, keep=keep, xf=xf, xm=xm, xp=xp, deg=deg,
                         b_row_ptr=bcsr.row_ptr, b_col_ind=bcsr.col_ind,
                         m_row_ptr=mcsr.row_ptr, m_col_ind=mcsr.col_ind).items():
            out[f"{name}/{k}"] = v
        out[f"{name}/src"] = np.array([src])
        big = n > 300
        for d in DIMS:
            p = f"{name}/d{d}"
            a = csr_to_b2sr(csr, d)
            at = b2sr_transpose(a)
            out[f"{p}/trp"], out[f"{p}/tci"], out[f"{p}/tiles"] = a.tile_row_ptr, a.tile_col_ind, a.bit_tiles
            out[f"{p}/t_trp"], out[f"{p}/t_tci"], out[f"{p}/t_tiles"] = (
                at.tile_row_ptr, at.tile_col_ind, at.bit_tiles)
            xbit = BitVector.from_bools(xb, d)
            kbit = BitVector.from_bools(keep, d)
            out[f"{p}/bbb"] = bmv_bin_bin_bin(a, xbit).words
            out[f"{p}/bbb_m"] = bmv_bin_bin_bin_masked(a, xbit, kbit).words
            out[f"{p}/bbf"] = bmv_bin_bin_full(a, xbit)
            out[f"{p}/bbf_m"] = bmv_bin_bin_full_masked(a, xbit, kbit)
            out[f"{p}/bff_ar"] = bmv_bin_full_full(a, xf, ARITHMETIC)
            out[f"{p}/bff_ar_m"] = bmv_bin_full_full_masked(a, xf, ARITHMETIC, kbit)
            out[f"{p}/bff_mp1"] = bmv_bin_full_full(a, xm, min_plus(1))
            out[f"{p}/bff_mp1_m"] = bmv_bin_full_full_masked(a, xm, min_plus(1), kbit)
            out[f"{p}/bff_mp0"] = bmv_bin_full_full(a, xm, min_plus(0))
            out[f"{p}/bff_mx"] = bmv_bin_full_full(a, xp, MAX_TIMES)
            out[f"{p}/used"] = used_columns(a)
            # scale with zeros only where no bits land (kernels.py:165-171)
            if n:
                sc = crng.uniform(0.5, 3.0, n)
                sc[~used_columns(a)] = 0.0
                out[f"{p}/scale"] = sc
                out[f"{p}/bff_sc"] = bmv_bin_full_full(a, xp, ARITHMETIC, scale=sc)
            b = csr_to_b2sr(bcsr, d)
            m = csr_to_b2sr(mcsr, d)
            out[f"{p}/bmm"] = np.array([bmm_bin_bin_sum(a, b)], np.int64)
            if not big or d <= 8:
                out[f"{p}/bmm_m"] = np.array([bmm_bin_bin_sum_masked(a, b, m)], np.int64)
                out[f"{p}/bmm_aa"] = np.array([bmm_bin_bin_sum_masked(a, a, a)], np.int64)
            r = bfs(a, src)
            out[f"{p}/bfs"], out[f"{p}/bfs_it"] = r.per_vertex, np.array([r.iterations])
            r = sssp(a, src)
            out[f"{p}/sssp"], out[f"{p}/sssp_it"] = r.per_vertex, np.array([r.iterations])
            r = pagerank(at, deg, AlgoParams())
            out[f"{p}/pr"], out[f"{p}/pr_it"] = r.per_vertex, np.array([r.iterations, int(r.converged)])
            if symmetric:
                r = connected_components(a)
                out[f"{p}/cc"], out[f"{p}/cc_it"] = r.per_vertex, np.array([r.iterations])
                if not big or d <= 8:
                    out[f"{p}/tc"] = np.array([triangle_count(csr, d).count], np.int64)
        manifest["cases"].append({"name": name, "n": n, "nnz": int(csr.nnz), "symmetric": symmetric})
        print(name, n, csr.nnz, flush=True)

    np.savez_compressed(HERE / "golden.npz", **out)
    (HERE / "manifest.json").write_text(json.dumps(manifest, indent=1) + "\n")
    print("wrote", HERE / "golden.npz", sum(v.nbytes for v in out.values()), "bytes raw")


if __name__ == "__main__":
    main()
