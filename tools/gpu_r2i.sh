set -x
for c in 0 1; do B2SR_CONV_SORT=$c timeout 600 python tools/conv_ab.py 22; done
B2SR_PR_TRACE=1 B2SR_PR_MODE=fast timeout 600 python tools/config4.py --scale 24 --no-oracle 2>&1 | grep -E "sweep [0-2] |pagerank" | cut -c1-300
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_rmat.py -q -x 2>&1 | tail -5
