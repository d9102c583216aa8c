set -x
O=gpurun_out
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'bfs|bmv|k_or|k_hot|k_live|k_row_live' --csv --log-file $O/r2bf_launch.csv python tools/bfs_probe.py --roots 16 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2bf_launch.csv 2>&1 | head -24
