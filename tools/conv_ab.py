"""csr_to_b2sr and b2sr_transpose timings (CUDA events, median of 3) at one
R-MAT scale, with algorithmic GB/s (SURVEY.md §8a bytes: CSR indices read +
B2SR written; transpose: B2SR read + written)."""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
dims = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8,16,32").split(",")]
csr = rmat.rmat_csr(scale, 16, seed=1)
n, nnz = csr.n, csr.nnz
out = {"scale": scale, "nnz": int(nnz)}
def timed(fn):
    ts, r = [], fn()  # warm: the memory pool grows on first use
    torch.cuda.synchronize()
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); r = fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    return r, sorted(ts)[1]
for d in dims:
    m, cms = timed(lambda: b2.csr_to_b2sr(csr, d))
    sb = b2.storage_bytes(m)
    t, tms = timed(lambda: b2.formats.B2srMatrix._wrap(b2.formats._new_handle("b2sr_transpose", m.handle().ptr, 0)))
    conv_bytes = 4 * (n + 1) + 4 * nnz + sb
    out[str(d)] = {"convert_ms": round(cms, 3), "convert_gbs": round(conv_bytes / cms / 1e6, 1),
                   "transpose_ms": round(tms, 3), "transpose_gbs": round(2 * sb / tms / 1e6, 1), "b2sr_bytes": sb}
    del m, t
    torch.cuda.empty_cache()
print(json.dumps(out))
