set -x
for r in 1 2; do for v in 1 2 3; do B2SR_BFS_LOOKAHEAD=$v timeout -s KILL 300 python tools/bfs_time.py 22 64; done; done
for v in 1 2; do B2SR_BFS_LOOKAHEAD=$v timeout -s KILL 300 python tools/bfs_time.py 20 64; done
for a in 2 4 8; do B2SR_BFS_ALPHA=$a timeout -s KILL 300 python tools/bfs_time.py 22 64; done
