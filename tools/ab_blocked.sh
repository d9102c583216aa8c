# A/B of the column-strip blocked kernels vs the row-major stream kernels
python -m pytest tests/test_gpu_rmat.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for B in 1 0; do
  B2SR_BLOCKED=$B python bench.py --steps 8 --warmup 2 --no-tc --no-cpu > gpurun_out/ab_$B.json 2> gpurun_out/ab_$B.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$B.json')); print('blocked=$B', 'bfs', d['value'], 'roof', d['roofline']['frac'], {k:(v['spmv_gbs'],v['spmv_frac'],v['bfs_ms']) for k,v in d['sweep'].items()})"
  tail -2 gpurun_out/ab_$B.err
done
