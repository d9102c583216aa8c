"""Triangle-count SpGEMM timing at one scale: count, kernel ms (CUDA events
around K8 on its stream), AND+POPC units.  Env B2SR_TC_HASH=0 selects the
binary-search items only (A/B)."""
import ctypes, json, sys, time
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import _capi, rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
dims = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "4,8").split(",")]
csr = rmat.rmat_csr(scale, 16, seed=1)
dag = b2.algorithms._degree_oriented(csr)
out = {"scale": scale}
for d in dims:
    lo = b2.csr_to_b2sr(dag, d)
    h = lo.handle()
    cnt, work = ctypes.c_int64(), ctypes.c_uint64()
    _capi.call("b2sr_tc_work", h.ptr, ctypes.addressof(cnt), ctypes.addressof(work), 0)
    b2.algorithms._tc_count(lo)
    ks = []
    _capi.call("b2sr_set_kernel_timing", 1)
    kms = ctypes.c_float()
    for _ in range(3):
        c = b2.algorithms._tc_count(lo)
        torch.cuda.synchronize()
        _capi.call("b2sr_last_kernel_ms", ctypes.addressof(kms))
        ks.append(kms.value)
    _capi.call("b2sr_set_kernel_timing", 0)
    out[str(d)] = {"triangles": c, "work_count": cnt.value, "kernel_ms": round(min(ks), 3), "units": work.value}
print(json.dumps(out))
