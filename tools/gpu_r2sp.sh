set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k 'upload or host or split' 2>&1 | tail -3
for r in 1 2; do
  for v in tiles split; do B2SR_H2D_PACK=$v timeout -s KILL 300 python tools/upload_probe.py 22; done
done
B2SR_H2D_THREADS=12 timeout -s KILL 300 python tools/upload_probe.py 22
B2SR_H2D_THREADS=15 timeout -s KILL 300 python tools/upload_probe.py 22
timeout -s KILL 300 python tools/upload_probe.py 24
B2SR_H2D_PACK=tiles timeout -s KILL 300 python tools/upload_probe.py 24
