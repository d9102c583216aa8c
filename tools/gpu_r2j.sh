set -x
O=gpurun_out
for p in 1 0; do B2SR_PR_XPERM=$p B2SR_PR_TRACE=1 B2SR_PR_MODE=fast timeout 600 python tools/config4.py --scale 24 --no-oracle 2>&1 | grep -E "sweep [0-2] |pagerank" | cut -c1-250; done
timeout 300 python tools/tc_ab.py 20 4,8
timeout 600 python tools/tc_ab.py 24 4
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_dist_native.py tests/test_acceptance_ports.py -q -x -k "bmm or tc or triangle or config2 or config3 or criterion" 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bfs.csv python tools/bfs_probe.py --scale 22 --dim 4 --roots 3 > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_bfs.csv 100 > $O/r02_launches_bfs_summary.txt; head -12 $O/r02_launches_bfs_summary.txt; grep -A80 "launch sequence" $O/r02_launches_bfs_summary.txt | tail -60
