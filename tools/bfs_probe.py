"""BFS at one scale / width for profiling: graph, transpose, a few roots
through b2sr_bfs (direction-optimizing, device-controlled)."""
import argparse, ctypes, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import _capi, rmat
from paper_2201_08560_b200 import _device as dev

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--dim", type=int, default=4)
ap.add_argument("--roots", type=int, default=3)
a = ap.parse_args()
csr = rmat.rmat_csr(a.scale, 16, seed=1)
deg = np.diff(csr.row_ptr.astype(np.int64))
m = b2.csr_to_b2sr(csr, a.dim)
at = b2.b2sr_transpose(m)
rng = np.random.default_rng(8)
roots = rng.choice(np.flatnonzero(deg > 0), size=a.roots, replace=False)
lv = dev.empty_bytes(8 * csr.n)
it = ctypes.c_int64()
for r in roots:
    _capi.call("b2sr_bfs", m.handle().ptr, at.handle().ptr, int(r), dev.ptr(lv), ctypes.addressof(it), dev.stream())
torch.cuda.synchronize()
print("sweeps", it.value)
