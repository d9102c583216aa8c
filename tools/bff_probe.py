"""Float-gather probe: one ARITHMETIC and one MINPLUS bmv_bin_full_full on R-MAT
at the given scale (for ncu), checked against the oracle when --check."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=20)
ap.add_argument("--dim", type=int, default=4)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--check", action="store_true")
a = ap.parse_args()
csr = rmat.rmat_csr(a.scale, 16, seed=1)
m = b2.csr_to_b2sr(csr, a.dim)
rng = np.random.default_rng(3)
x = rng.random(csr.n)
import ctypes
from paper_2201_08560_b200 import _capi
from paper_2201_08560_b200 import _device as dev
h = m.handle()
xd = dev.to_device(x)
yd = dev.empty_bytes(8 * csr.n)
bad = ctypes.c_int64(-1)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(a.reps):
    ts = []
    for ring, inc in ((1, 0.0), (2, 1.0)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _capi.call("b2sr_bmv_bff", h.ptr, dev.ptr(xd), ring, inc, None, None, dev.ptr(yd), ctypes.addressof(bad), sp)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"device: arith {ts[0]:.3f} ms  minplus {ts[1]:.3f} ms", flush=True)
ya = b2.bmv_bin_full_full(m, x, b2.ARITHMETIC)
yb = b2.bmv_bin_full_full(m, x, b2.min_plus(1))
if a.check:
    from oracle import oracle as orc
    ref = (csr.n, a.dim, m.tile_row_ptr, m.tile_col_ind, m.bit_tiles)
    ra = orc.bmv_bff(ref, x, "arithmetic", workers=16)
    rb = orc.bmv_bff(ref, x, "minplus", 1.0, workers=16)
    print("arith equal", ya.tobytes() == ra.tobytes(), "minplus equal", yb.tobytes() == rb.tobytes())
    bad = np.flatnonzero(yb != rb)
    print("minplus mismatches", len(bad), bad[:5], yb[bad[:5]], rb[bad[:5]])
if a.scale >= 23:  # vertex term-count profile of the segmented plan rows
    deg = np.diff(csr.row_ptr.astype(np.int64))
    print("deg>2048:", int((deg > 2048).sum()), "terms", int(deg[deg > 2048].sum()), "max", int(deg.max()))
