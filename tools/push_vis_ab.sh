# A/B: visited filter in the direction-optimizing push levels x alpha (BFS s22 d=4)
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "algorithms or rmat or hot" 2>&1 | tail -1
for V in 0 1; do for a in 2 4 8 16 32; do
  B2SR_PUSH_VISITED=$V B2SR_BFS_ALPHA=$a timeout 600 python bench.py --steps 32 --warmup 3 --dims 4 --dim 4 --no-cpu --no-tc --no-drivers 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('vis $V alpha $a', d['value'], d['ms_per_step'])"
done; done
