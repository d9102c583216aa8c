cat > /tmp/tcprobe.py <<'PY'
import sys; sys.path.insert(0, '.')
import paper_2201_08560_b200 as b2
from paper_2201_08560_b200 import rmat
csr = rmat.rmat_csr(20, 16, seed=1)
lo = b2.csr_to_b2sr(b2.algorithms._degree_oriented(csr), 4)
for _ in range(2): print(b2.algorithms._tc_count(lo))
PY
timeout 600 ncu --set full --import-source on -k regex:bmm_masked -s 1 -c 1 -o gpurun_out/ncu_tc python /tmp/tcprobe.py > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/ncu_tc.ncu-rep | grep -E "time_dur|inst_exec|issue_active|stalls"
