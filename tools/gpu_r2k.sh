set -x
O=gpurun_out
timeout 900 python bench.py --no-tc --no-drivers --no-config5 --no-cpu --dims 4 > $O/bench_bfs.json 2> $O/bench_bfs.err; echo rc=$?
python -c "import json;d=json.loads(open('$O/bench_bfs.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d.get('gteps_harmonic_mean'),d['bfs_bytes'])"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bfs2.csv python tools/bfs_probe.py --scale 22 --dim 4 --roots 3 > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_bfs2.csv | grep -E "bfs|total"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py tests/test_gpu_dist_native.py -q -x -k "bfs or sssp" 2>&1 | tail -3
