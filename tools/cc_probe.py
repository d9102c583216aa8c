"""connected_components at one R-MAT scale (d=4): CUDA-event time of the
whole call (median of 3 after a warm call) and the sweep count."""
import json, sys
from pathlib import Path
import torch
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
m = b2.csr_to_b2sr(rmat.rmat_csr(scale, 16, seed=1), 4)
r = b2.connected_components(m)
ts = []
for _ in range(reps):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); r = b2.connected_components(m); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"scale": scale, "cc_ms": round(sorted(ts)[len(ts) // 2], 3), "iterations": r.iterations}))
