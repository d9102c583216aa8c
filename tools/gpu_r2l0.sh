set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py tests/test_gpu_dist_native.py tests/test_acceptance_ports.py -q -x -p no:cacheprovider -k 'bfs or algorithms or rmat or worked or hot or push or sssp or errors or concurrent' 2>&1 | tail -3
for r in 1 2 3; do timeout -s KILL 300 python tools/bfs_time.py 22 64; done
timeout -s KILL 300 python tools/bfs_time.py 20 64
timeout -s KILL 300 python tools/push_probe.py --scale 22 --dims 4 --roots 8 2>&1 | tail -1
