set -x
for t in 4 8 12 16; do for p in 1 0; do B2SR_H2D_THREADS=$t B2SR_H2D_PACK=$p timeout -s KILL 120 python tools/upload_probe.py | tail -1; done; done
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k "conversion or large_host or roundtrip or profile" 2>&1 | tail -1
timeout -s KILL 200 python tools/conv_ab.py 22 4,8
B2SR_CONV_COUNT=merge timeout -s KILL 200 python tools/conv_ab.py 22 4,8
