# BFS changes + x-gather cache-policy A/B for the K4 stream kernel
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for XG in 0 1 2; do
  B2SR_XGATHER=$XG python bench.py --steps 8 --warmup 2 --no-tc --no-cpu > gpurun_out/xg_$XG.json 2> gpurun_out/xg_$XG.err
  python -c "import json; d=json.load(open('gpurun_out/xg_$XG.json')); print('xg=$XG', 'bfs', d['value'], 'roof', d['roofline']['frac'], {k:(v['spmv_gbs'],v['spmv_frac'],v['bfs_ms']) for k,v in d['sweep'].items()}, d['e2e'].get('breakdown_ms'))"
  tail -2 gpurun_out/xg_$XG.err
done
B2SR_BFS_TRACE=1 python bench.py --steps 2 --warmup 1 --dims 4 --dim 4 --no-tc --no-cpu 2>&1 | grep "b2sr bfs" | head -9
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bfs|active" -c 200 --csv --log-file gpurun_out/launches_bfs3.csv python bench.py --steps 2 --warmup 1 --dims 4 --dim 4 --no-tc --no-cpu > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_bfs3.csv 30
