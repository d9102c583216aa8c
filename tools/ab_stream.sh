timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -x -q 2>&1 | tail -3
for V in "B2SR_STREAM=0" "B2SR_STREAM=1"; do
  env $V timeout 600 python bench.py --steps 8 --warmup 3 --dims 4,8 --no-cpu --no-drivers --no-tc > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$V', 'bfs', d['value'], 'roof', d['roofline']['frac'], {k:(v['spmv_gbs'],v['spmv_frac'],v['bfs_ms'],v['bfs_gteps']) for k,v in d['sweep'].items()})" || tail -3 gpurun_out/ab.err
done
