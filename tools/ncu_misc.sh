# ncu --set full summaries of the other hot kernels (profiles/r01_ncu_misc.txt):
# K8 masked SpGEMM (TC s20 d=4), the push-only BFS level, CC's u32 minimum (s24),
# and K7's gather
mkdir -p gpurun_out
cat > /tmp/tcprobe.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat
csr = rmat.rmat_csr(20, 16, seed=1)
lo = b2.csr_to_b2sr(b2.algorithms._degree_oriented(csr), 4)
for _ in range(2): print(b2.algorithms._tc_count(lo))
m = b2.csr_to_b2sr(csr, 4)
print(b2.bmm_bin_bin_sum(m, m))
for r in (1, 2): b2.bfs(b2.csr_to_b2sr(csr, 4), r)   # fresh matrices: push-only levels
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bmm_masked_items|k_bmm_sum_gather|k_bfs_push_level" -c 8 -o gpurun_out/ncu_misc python /tmp/tcprobe.py > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_cc_min" -c 1 -o gpurun_out/ncu_cc python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/ncu_misc.ncu-rep > gpurun_out/ncu_misc.txt
python tools/ncu_kv.py gpurun_out/ncu_cc.ncu-rep >> gpurun_out/ncu_misc.txt
grep -E "==|time_dur|dram__bytes_read|issue_active" gpurun_out/ncu_misc.txt | head -60
