# A/B of the hot-column smem x cache (hot.cu) + flat stream K4 (bmv_stream.cu)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for V in "B2SR_HOT=0" "B2SR_STREAM=0" "B2SR_STREAM=1"; do
  env $V timeout 600 python bench.py --steps 16 --warmup 3 --dims 4,8,16 --no-cpu --no-drivers --no-tc > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('$V', 'bfs', d['value'], 'roof', d['roofline']['frac'], {k:(v['spmv_gbs'],v['spmv_frac'],v['bfs_ms'],v['bfs_gteps']) for k,v in d['sweep'].items()})" || tail -3 gpurun_out/ab.err
done
