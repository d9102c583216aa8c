# parity tests; BFS pull variants; TC kernels; float-gather profile at s24
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for PV in group warp; do
  B2SR_PULL=$PV python bench.py --steps 8 --warmup 2 --dims 4,8 --no-cpu --no-drivers > gpurun_out/pull_$PV.json 2> gpurun_out/pull_$PV.err
  python -c "import json; d=json.load(open('gpurun_out/pull_$PV.json')); print('pull=$PV', 'bfs', d['value'], {k:(v['bfs_ms'],v['bfs_gteps']) for k,v in d['sweep'].items()}, 'tc', {k:v['ms'] for k,v in d['tc']['by_tile_dim'].items()}, 'e2e', d['e2e']['breakdown_ms'])"
  tail -2 gpurun_out/pull_$PV.err
done
B2SR_TC_ALG=items python bench.py --steps 2 --warmup 1 --dims 4 --dim 4 --no-cpu --no-drivers 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tc items', {k:(v['ms'],v['triangles']) for k,v in d['tc']['by_tile_dim'].items()})"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bff|pr_|pw_|relax|cc_" -c 120 --csv --log-file gpurun_out/launches_pr.csv python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_pr.csv 40
