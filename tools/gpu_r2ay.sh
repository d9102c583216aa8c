set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k "conversion or roundtrip or profile or rmat_against or large_host" 2>&1 | tail -1
for i in 1 2; do timeout -s KILL 200 python tools/conv_ab.py 22 4,8; done
