"""Device-resident BFS timing at one scale (d=4, direction-optimizing,
device-controlled): ms per root over R roots after a warm-up (CUDA events),
as the bench's headline loop does, without the rest of the bench."""
import ctypes, json, sys
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import _capi, rmat
from paper_2201_08560_b200 import _device as dev

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
R = int(sys.argv[2]) if len(sys.argv) > 2 else 64
csr = rmat.rmat_csr(scale, 16, seed=1)
deg = np.diff(csr.row_ptr.astype(np.int64))
m = b2.csr_to_b2sr(csr, 4)
at = b2.b2sr_transpose(m)
rng = np.random.default_rng(8)
roots = rng.choice(np.flatnonzero(deg > 0), size=R + 4, replace=False)
lv = dev.empty_bytes(8 * csr.n)
it = ctypes.c_int64()
run = lambda r: _capi.call("b2sr_bfs", m.handle().ptr, at.handle().ptr, int(r), dev.ptr(lv), ctypes.addressof(it), dev.stream())
for r in roots[:4]:
    run(r)
torch.cuda.synchronize()
res = []
for rep in range(3):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for r in roots[4:]:
        run(r)
    b.record(); torch.cuda.synchronize()
    res.append(a.elapsed_time(b) / R)
print(json.dumps({"scale": scale, "roots": R, "ms_per_root": [round(x, 4) for x in res]}))
