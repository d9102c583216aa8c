timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 300 python tools/spmv_probe.py --reps 8 --dims 4,8
timeout 600 python bench.py --steps 32 --warmup 3 --dims 4 --dim 4 --no-cpu --no-drivers --no-tc | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bfs', d['value'], 'roof', d['roofline']['frac'])"
