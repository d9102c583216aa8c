set -x
for r in 1 2; do for v in 1 2 4; do B2SR_BFS_UPD_CHUNKS=$v timeout -s KILL 300 python tools/bfs_time.py 22 64; done; done
for v in 1 2 4; do B2SR_BFS_UPD_CHUNKS=$v timeout -s KILL 300 python tools/bfs_time.py 20 64; done
