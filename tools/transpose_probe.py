import sys, time; sys.path.insert(0, '.')
import torch
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat
csr = rmat.rmat_csr(22, 16, seed=1)
m = b2.csr_to_b2sr(csr, 4)
for i in range(3):
    m._transpose = None
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); t = b2.b2sr_transpose(m); e1.record(); torch.cuda.synchronize()
    print("transpose ms", e0.elapsed_time(e1))
