set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tc or triangle or masked_spgemm or bmm" 2>&1 | tail -1
timeout -s KILL 300 python tools/tc_ab.py 20 4,8
timeout -s KILL 600 python tools/tc_ab.py 26 4
