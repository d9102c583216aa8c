set -x
O=gpurun_out
lscpu | head -20 > $O/r2nt_lscpu.txt; nproc >> $O/r2nt_lscpu.txt
timeout -s KILL 600 python -m pytest tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k 'upload or host' 2>&1 | tail -2
for r in 1 2; do
  for v in 0 1; do B2SR_H2D_NT=$v timeout -s KILL 300 python tools/upload_probe.py 22; done
done
B2SR_H2D_NT=1 B2SR_H2D_PACK=all timeout -s KILL 300 python tools/upload_probe.py 22
B2SR_H2D_NT=1 B2SR_H2D_PACK=0 timeout -s KILL 300 python tools/upload_probe.py 22
B2SR_H2D_NT=0 B2SR_H2D_PACK=0 timeout -s KILL 300 python tools/upload_probe.py 22
