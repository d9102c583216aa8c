set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'algorithms or worked' 2>&1 | tail -2
for r in 1 2; do for v in 256 128 64; do B2SR_BFS_UPD_THREADS=$v timeout -s KILL 300 python tools/bfs_time.py 22 64; done; done
for v in 256 128 64; do B2SR_BFS_UPD_THREADS=$v timeout -s KILL 300 python tools/bfs_time.py 20 64; done
