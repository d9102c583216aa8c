set -x
for r in 1 2; do for v in 8 4 2 1; do B2SR_BFS_PREP_CTAS=$v timeout -s KILL 300 python tools/bfs_time.py 22 64; done; done
for v in 8 2; do B2SR_BFS_PREP_CTAS=$v timeout -s KILL 300 python tools/bfs_time.py 20 64; done
