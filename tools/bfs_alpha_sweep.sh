set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "algorithms or worked or rmat" 2>&1 | tail -3
for a in 2 4 8 16; do B2SR_BFS_ALPHA=$a python bench.py --steps 8 --warmup 2 --dims 4,8 --no-tc --no-cpu 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('alpha', $a, d['value'], d['ms_per_step'], {k:(v['bfs_ms'],v['bfs_gteps']) for k,v in d['sweep'].items()})"; done
B2SR_BFS_TRACE=1 python bench.py --steps 2 --warmup 1 --dims 4 --dim 4 --no-tc --no-cpu 2>&1 | grep "b2sr bfs" | head -20
