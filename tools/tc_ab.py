import sys, os, time; sys.path.insert(0, '.')
import torch
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat
csr = rmat.rmat_csr(20, 16, seed=1)
for orient in ("id", "degree"):
    L = b2.algorithms._degree_oriented(csr) if orient == "degree" else b2.lower_triangle(csr)
    for d in (4, 8):
        lo = b2.csr_to_b2sr(L, d)
        c = b2.algorithms._tc_count(lo); torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); c = b2.algorithms._tc_count(lo); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
        print(orient, d, c, round(min(ts), 2), "ms", flush=True)
