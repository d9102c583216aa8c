set -x
O=gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py tests/test_gpu_dist_native.py -q -x -p no:cacheprovider -k 'bfs or algorithms or rmat or worked or hot' 2>&1 | tail -3
for r in 1 2 3; do for v in 0 1; do B2SR_BFS_PDL=$v timeout -s KILL 300 python tools/bfs_time.py 22 64; done; done
for v in 0 1; do B2SR_BFS_PDL=$v timeout -s KILL 300 python tools/bfs_time.py 20 64; done
