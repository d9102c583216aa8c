set -x
for r in 1 2; do for v in 8 12 16; do B2SR_BFS_PREP_CTAS=$v timeout -s KILL 300 python tools/bfs_time.py 22 64; done; done
