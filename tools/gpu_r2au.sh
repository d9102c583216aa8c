set -x
O=gpurun_out
for la in 1 2 3 4; do for r in 1 2; do B2SR_BFS_LOOKAHEAD=$la timeout -s KILL 600 python bench.py --no-config5 --no-drivers --no-tc --no-cpu --dims 4 > $O/r2au.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/r2au.json').read().strip().splitlines()[-1]);print('la=$la', d['value'],d['ms_per_step'],d['sweep']['4']['bfs_gteps'])"; done; done
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bfs or algorithms" 2>&1 | tail -1
