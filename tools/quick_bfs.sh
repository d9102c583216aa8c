timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -x -q 2>&1 | tail -2
for V in "B2SR_BFS_DEVCTL=0" "B2SR_BFS_DEVCTL=1"; do
  env $V timeout 600 python bench.py --steps 16 --warmup 3 --dims 4,8 --no-cpu --no-drivers --no-tc > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$V', 'bfs', d['value'], d['config']['tile_dim'], 'roof', d['roofline']['frac'], {k:(v['spmv_gbs'],v['spmv_frac'],v['bfs_ms'],v['bfs_gteps']) for k,v in d['sweep'].items()}, d['e2e']['breakdown_ms'])" || tail -3 gpurun_out/ab.err
done
B2SR_BFS_TRACE=1 timeout 300 python bench.py --steps 2 --warmup 1 --dims 4 --dim 4 --no-cpu --no-drivers --no-tc 2>&1 >/dev/null | tail -9
