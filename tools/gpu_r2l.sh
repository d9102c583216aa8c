set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py tests/test_gpu_dist_native.py -q -x -k "bfs or sssp" 2>&1 | tail -3
bash tools/sanitize.sh
