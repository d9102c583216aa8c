set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k 'conversion or rmat or random or roundtrip or upload' 2>&1 | tail -3
for r in 1 2; do timeout -s KILL 300 python tools/conv_ab.py 22 4,8,16; done
timeout -s KILL 300 python tools/conv_ab.py 24 4
