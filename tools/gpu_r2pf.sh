set -x
O=gpurun_out
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:k_bmv_bbb_stream -c 1 -o $O/r02_ncu_k4_v9 python tools/spmv_probe.py --dims 4 --reps 2 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_k4_v9.ncu-rep > $O/r2pf_k4.txt 2>&1
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:k_bfs_level -s 4 -c 4 -o $O/r02_ncu_bfs_level_v9 python tools/bfs_time.py 22 2 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_bfs_level_v9.ncu-rep > $O/r2pf_bfs.txt 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2pf_bfs_launch.csv python tools/bfs_time.py 22 16 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2pf_bfs_launch.csv > $O/r2pf_bfs_launch.txt 2>&1
