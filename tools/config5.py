"""BASELINE configs[4] on one GPU: BFS and triangle counting on R-MAT scale 26.

    python tools/config5.py [--scale 26] [--roots 8]
Prints one JSON line (BFS GTEPS over a few Graph500 roots, TC time and count).
The multi-GPU runs of this config go through bench.py under torchrun."""
import argparse
import ctypes
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2  # noqa: E402
from paper_2201_08560_b200 import _capi, rmat  # noqa: E402
from paper_2201_08560_b200 import _device as dev  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=26)
    ap.add_argument("--roots", type=int, default=8)
    ap.add_argument("--check-lower", action="store_true",
                    help="also count on the ID-ordered lower triangle (the reference's L): same count expected")
    a = ap.parse_args()
    torch.cuda.set_device(0)
    t0 = time.time()
    csr = rmat.rmat_csr(a.scale, 16, seed=1)
    gen = time.time() - t0
    n = csr.n
    deg = np.diff(csr.row_ptr.astype(np.int64))
    out = {"config": f"R-MAT scale {a.scale} undirected, B2SR-4, one GPU", "n": n, "nnz": int(csr.nnz),
           "graph_gen_s": round(gen, 2)}
    # TC first (the DAG and its B2SR are freed before the BFS matrices are built)
    t0 = time.time()
    dag = b2.algorithms._degree_oriented(csr)
    lo = b2.csr_to_b2sr(dag, 4)
    del dag
    torch.cuda.synchronize()
    setup = time.time() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tri = b2.algorithms._tc_count(lo)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    out["tc"] = {"triangles": int(tri), "ms": round(ms, 2), "edges_per_s": round((csr.nnz // 2) / (ms / 1e3), 1),
                 "dag_tiles": int(lo.num_tiles), "setup_s": round(setup, 2)}
    del lo
    torch.cuda.empty_cache()
    if a.check_lower:  # orientation invariance at a scale the reference cannot run
        lo = b2.csr_to_b2sr(b2.lower_triangle(csr), 4)
        e0.record()
        tri2 = b2.algorithms._tc_count(lo)
        e1.record()
        torch.cuda.synchronize()
        out["tc"]["lower_triangle_count"] = int(tri2)
        out["tc"]["lower_triangle_ms"] = round(e0.elapsed_time(e1), 2)
        out["tc"]["counts_equal"] = int(tri2) == int(tri)
        del lo
        torch.cuda.empty_cache()
    m = b2.csr_to_b2sr(csr, 4)
    at = b2.b2sr_transpose(m)
    rng = np.random.default_rng(8)
    roots = [int(v) for v in rng.choice(np.flatnonzero(deg > 0), size=a.roots + 1, replace=False)]
    lv = dev.empty_bytes(8 * n)
    it = ctypes.c_int64()
    sp = torch.cuda.current_stream().cuda_stream
    _capi.call("b2sr_bfs", m.handle().ptr, at.handle().ptr, roots[0], dev.ptr(lv), ctypes.addressof(it), sp)
    degt = torch.from_numpy(deg).to("cuda")
    edges, tot = 0, 0.0
    for r in roots[1:]:
        e0.record()
        _capi.call("b2sr_bfs", m.handle().ptr, at.handle().ptr, r, dev.ptr(lv), ctypes.addressof(it), sp)
        e1.record()
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
        edges += int(degt[torch.isfinite(lv.view(torch.float64)[:n])].sum().item()) // 2
    out["bfs"] = {"roots": a.roots, "ms_per_root": round(tot / a.roots, 3), "gteps": round(edges / (tot / 1e3) / 1e9, 2)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
