"""Host-matrix upload (b2sr_from_host via B2srMatrix.handle()) of R-MAT s22
B2SR-4 host arrays: median of 5, ms and GB/s of host bytes.  Knobs:
B2SR_H2D_THREADS, B2SR_H2D_PACK=0."""
import json, os, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
csr = rmat.rmat_csr(scale, 16, seed=1)
m = b2.csr_to_b2sr(csr, 4)
host = (m.tile_row_ptr.copy(), m.tile_col_ind.copy(), m.bit_tiles.copy())
nb = sum(a.nbytes for a in host)
del m
torch.cuda.empty_cache()
ts = []
for i in range(6):
    hm = b2.B2srMatrix(csr.n, 4, *host)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); h = hm.handle(); e1.record(); torch.cuda.synchronize()
    if i:
        ts.append(e0.elapsed_time(e1))
    del h, hm
ms = float(np.median(ts))
print(json.dumps({"threads": os.environ.get("B2SR_H2D_THREADS", "default"), "pack": os.environ.get("B2SR_H2D_PACK", "1"),
                  "ms": round(ms, 2), "host_GBs": round(nb / ms / 1e6, 1), "bytes": nb}))
