timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -x -q 2>&1 | tail -2
for V in "B2SR_BFS_HEAD=0" "B2SR_BFS_HEAD=1"; do
env $V timeout 600 python bench.py --steps 64 --warmup 3 --dims 4 --dim 4 --no-cpu --no-drivers --no-tc > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$V bfs', d['value'], d['ms_per_step'])" || tail -3 gpurun_out/ab.err
done
