"""Push-only BFS (no transpose) vs transpose + direction-optimizing BFS on R-MAT:
per-root device times and level parity between the two paths."""
import argparse, ctypes, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat, _capi
from paper_2201_08560_b200 import _device as dev

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--dims", default="4,8")
ap.add_argument("--roots", type=int, default=6)
a = ap.parse_args()
csr = rmat.rmat_csr(a.scale, 16, seed=1)
n = csr.n
deg = np.diff(csr.row_ptr.astype(np.int64))
roots = np.random.default_rng(7).choice(np.flatnonzero(deg > 0), a.roots, replace=False)
sp = torch.cuda.current_stream().cuda_stream
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
for d in map(int, a.dims.split(",")):
    m = b2.csr_to_b2sr(csr, d)
    hA = m.handle()
    torch.cuda.synchronize()
    e0, e1 = ev(), ev()
    e0.record()
    at = b2.b2sr_transpose(m)
    hT = at.handle()
    e1.record()
    torch.cuda.synchronize()
    tr_ms = e0.elapsed_time(e1)
    it = ctypes.c_int64()
    la, lb = dev.empty_bytes(8 * n), dev.empty_bytes(8 * n)
    res = {"push": [], "dopt": []}
    for k, r in enumerate(roots):
        for name, ht, buf in (("push", None, la), ("dopt", hT.ptr, lb)):
            e0, e1 = ev(), ev()
            e0.record()
            _capi.call("b2sr_bfs", hA.ptr, ht, int(r), dev.ptr(buf), ctypes.addressof(it), sp)
            e1.record()
            torch.cuda.synchronize()
            res[name].append((e0.elapsed_time(e1), int(it.value)))
        same = torch.equal(la.view(torch.float64)[:n], lb.view(torch.float64)[:n])
        print(f"d={d} root {r}: push {res['push'][-1]} dopt {res['dopt'][-1]} equal={same}", flush=True)
    pm = np.mean([t for t, _ in res["push"][1:]])
    dm = np.mean([t for t, _ in res["dopt"][1:]])
    print(f"d={d}: transpose {tr_ms:.3f} ms, push-only {pm:.3f} ms/root, dopt {dm:.3f} ms/root "
          f"(first calls {res['push'][0][0]:.3f} / {res['dopt'][0][0]:.3f})", flush=True)
    del hA, hT, m, at
    torch.cuda.empty_cache()
