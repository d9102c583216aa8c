timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -x -q 2>&1 | tail -1
timeout 600 python bench.py --steps 64 --warmup 3 --dims 4 --dim 4 --no-cpu --no-drivers --no-tc | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bfs', d['value'], d['ms_per_step'], d['bfs_sweeps_per_root'])"
