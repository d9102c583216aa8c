"""K4 bbb probe: R-MAT s22 masked sweep at the given widths (for ncu / A-B)."""
import argparse, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np, torch
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import _capi, rmat
from paper_2201_08560_b200 import _device as dev

ap = argparse.ArgumentParser()
ap.add_argument("--scale", type=int, default=22)
ap.add_argument("--dims", default="4,8")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
csr = rmat.rmat_csr(a.scale, 16, seed=1)
n = csr.n
rng = np.random.default_rng(11)
sp = torch.cuda.current_stream().cuda_stream
for d in [int(x) for x in a.dims.split(",")]:
    m = b2.csr_to_b2sr(csr, d)
    h = m.handle()
    ntr = h.ntr
    xd = dev.to_device(b2.BitVector.from_bools(rng.random(n) < 0.5, d).words, dev.padded_vec_bytes(ntr, d))
    kd = dev.to_device(b2.BitVector.from_bools(rng.random(n) < 0.5, d).words, dev.padded_vec_bytes(ntr, d))
    yd = dev.empty_bytes(dev.padded_vec_bytes(ntr, d))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for i in range(a.reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        _capi.call("b2sr_bmv_bbb", h.ptr, dev.ptr(xd), dev.ptr(kd), dev.ptr(yd), sp)
        e1.record()
        torch.cuda.synchronize()
        if i:
            ts.append(e0.elapsed_time(e1))
    wb = 4 if d == 32 else (2 if d == 16 else 1)
    ab = 4 * (ntr + 1) + h.num_tiles * (4 + d * wb) + 3 * ntr * wb
    if ts:
        ms = float(np.mean(ts))
        print(f"d {d} tiles {h.num_tiles} bbb {ms:.4f} ms {ab / ms / 1e6:.1f} GB/s", flush=True)
