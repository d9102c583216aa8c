# CLI on BASELINE configs[0] (R-MAT s16, d=32) and s18 d=4: bench every kernel
# against cuSPARSE CSR on the same GPU; reports under gpurun_out/cli/.
set -e
mkdir -p gpurun_out/cli
python - <<'PY'
import numpy as np, sys
sys.path.insert(0, ".")
from oracle import oracle as orc
for s in (16, 18):
    rp, ci = orc.rmat_csr(s, 16, seed=1)
    n = len(rp) - 1
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp.astype(np.int64))) + 1
    with open(f"gpurun_out/cli/rmat{s}.mtx", "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate pattern general\n")
        fh.write(f"{n} {n} {len(ci)}\n")
        np.savetxt(fh, np.stack([rows, ci.astype(np.int64) + 1], 1), fmt="%d")
PY
for k in bmv-bbb bmv-bbf bmv-bff bmm-sum; do
  timeout 600 python -m paper_2201_08560_b200.cli bench gpurun_out/cli/rmat16.mtx --kernel $k --tile-dim 32 --reps 5 --json gpurun_out/cli/bench16_$k.json | tail -3
  timeout 600 python -m paper_2201_08560_b200.cli bench gpurun_out/cli/rmat18.mtx --kernel $k --tile-dim 4 --reps 5 --json gpurun_out/cli/bench18_$k.json | tail -3
done
timeout 600 python -m paper_2201_08560_b200.cli profile gpurun_out/cli/rmat18.mtx --json gpurun_out/cli/profile18.json | tail -2
timeout 600 python -m paper_2201_08560_b200.cli run bfs gpurun_out/cli/rmat18.mtx --src 1 --json gpurun_out/cli/run18_bfs.json | head -2
timeout 600 python -m paper_2201_08560_b200.cli run tc gpurun_out/cli/rmat18.mtx --tile-dim 4 --json gpurun_out/cli/run18_tc.json | head -3
rm -f gpurun_out/cli/*.mtx
