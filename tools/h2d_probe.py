"""H2D rates for a 1 GB upload: pageable torch copy_, page-locked copy_, and
the library's staged b2sr_h2d from pageable numpy (staging.cu)."""
import sys, time, json
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2201_08560_b200 import _capi

nb = 1 << 30
a = np.random.default_rng(0).integers(0, 255, nb, dtype=np.uint8)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
pin = torch.empty(nb, dtype=torch.uint8, pin_memory=True); pin.numpy()[:] = a
s = torch.cuda.current_stream().cuda_stream
out = {}
def rate(fn, reps=4):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
    return round(nb / min(ts) / 1e9, 2)
out["pageable_copy_GBs"] = rate(lambda: d.copy_(torch.from_numpy(a)))
out["pinned_copy_GBs"] = rate(lambda: d.copy_(pin, non_blocking=True))
out["staged_b2sr_h2d_GBs"] = rate(lambda: _capi.call("b2sr_h2d", d.data_ptr(), a.ctypes.data, nb, s))
assert torch.equal(d.cpu(), torch.from_numpy(a))
print(json.dumps(out))
# register-in-place: cudaHostRegister the caller's pages, DMA, unregister
# (whole buffer, and in 64 MB pieces), to see whether pinning beats the staging memcpy
cr = torch.cuda.cudart()
def reg_whole():
    assert cr.cudaHostRegister(a.ctypes.data, nb, 0) == 0
    d.copy_(torch.from_numpy(a), non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(a.ctypes.data)
t0 = time.perf_counter(); assert cr.cudaHostRegister(a.ctypes.data, nb, 0) == 0; t1 = time.perf_counter()
cr.cudaHostUnregister(a.ctypes.data); t2 = time.perf_counter()
out["register_1GB_ms"] = round((t1 - t0) * 1e3, 2)
out["unregister_1GB_ms"] = round((t2 - t1) * 1e3, 2)
out["register_copy_unregister_GBs"] = rate(reg_whole)
nproc = os.cpu_count() if False else None
import os
out["cpu_count"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
print(json.dumps(out))
