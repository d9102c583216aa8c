"""BASELINE configs[3]: PageRank, SSSP (min-plus) and CC on R-MAT scale 24.

Runs the device drivers through the public API, times them with CUDA events,
then checks them against the C oracle (restated reference loops, OpenMP) on
the same graph -- the reference itself cannot run at this scale (its
transpose needs ~16*d^2 bytes per tile).  Because the graph is undirected and
loop-free, the oracle gets the matrix as its own transpose (SURVEY.md §8c
restatement rule), so its setup cost is not part of its timing either.

    python tools/config4.py [--scale 24] [--dim 4] [--no-oracle]
Writes one JSON line to stdout.
"""

import argparse
import ctypes
import json
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2  # noqa: E402
from paper_2201_08560_b200 import rmat  # noqa: E402


def ev():
    return torch.cuda.Event(enable_timing=True)


def timed(fn):
    a, b = ev(), ev()
    a.record()
    out = fn()
    b.record()
    torch.cuda.synchronize()
    return out, a.elapsed_time(b)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--dim", type=int, default=4)
    ap.add_argument("--no-oracle", action="store_true")
    args = ap.parse_args()
    torch.cuda.set_device(0)
    t0 = time.time()
    csr = rmat.rmat_csr(args.scale, 16, seed=1)
    n = csr.n
    m = b2.csr_to_b2sr(csr, args.dim)
    at = b2.b2sr_transpose(m)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    deg = np.diff(csr.row_ptr.astype(np.int64)).astype(np.float64)
    src = int(np.argmax(deg))
    out = {"config": f"R-MAT scale {args.scale} undirected, B2SR-{args.dim}", "n": n, "nnz": int(csr.nnz),
           "tiles": int(m.num_tiles), "b2sr_bytes": int(b2.storage_bytes(m)), "setup_s": round(setup_s, 2)}
    b2.pagerank(at, deg)  # warm (work partition, pairwise tree)
    pr, ms = timed(lambda: b2.pagerank(at, deg))
    out["pagerank"] = {"ms": round(ms, 3), "iterations": pr.iterations, "ms_per_iter": round(ms / pr.iterations, 3)}
    b2.sssp(m, src)
    ss, ms = timed(lambda: b2.sssp(m, src))
    out["sssp"] = {"ms": round(ms, 3), "iterations": ss.iterations, "src": src}
    b2.connected_components(m)
    cc, ms = timed(lambda: b2.connected_components(m))
    out["cc"] = {"ms": round(ms, 3), "iterations": cc.iterations,
                 "components": int(len(np.unique(cc.per_vertex)))}
    if not args.no_oracle:
        from oracle import oracle as orc

        threads = os.cpu_count() or 1
        L = orc.lib()
        ref = (n, args.dim, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles)
        P = ctypes.c_void_p
        arr = [ref[2].ctypes.data, ref[3].ctypes.data, np.ascontiguousarray(ref[4]).ctypes.data]
        t = time.perf_counter()
        rank = np.zeros(n)
        conv, bad = ctypes.c_int(), ctypes.c_int64()
        it = L.orc_pagerank(n, args.dim, *arr, deg.ctypes.data, 0.85, 1e-9, 10, rank.ctypes.data,
                            ctypes.addressof(conv), ctypes.addressof(bad), threads)
        out["pagerank"].update(oracle_s=round(time.perf_counter() - t, 2), oracle_iterations=int(it),
                               bitwise_equal=rank.tobytes() == pr.per_vertex.tobytes(),
                               rel_l1=float(np.abs(rank - pr.per_vertex).sum() / np.abs(rank).sum()))
        t = time.perf_counter()
        dist = np.zeros(n)
        it = L.orc_sssp(n, args.dim, *arr, src, dist.ctypes.data, threads)
        out["sssp"].update(oracle_s=round(time.perf_counter() - t, 2), oracle_iterations=int(it),
                           bitwise_equal=dist.tobytes() == ss.per_vertex.tobytes())
        t = time.perf_counter()
        lab = np.zeros(n)
        it = L.orc_cc(n, args.dim, *arr, lab.ctypes.data, threads)
        out["cc"].update(oracle_s=round(time.perf_counter() - t, 2), oracle_iterations=int(it),
                         bitwise_equal=lab.tobytes() == cc.per_vertex.tobytes())
        out["oracle_threads"] = threads
        del P
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
