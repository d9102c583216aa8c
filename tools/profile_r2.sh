# round-2 ncu evidence (profiles/r02_*): launch list of a short default bench,
# full captures of the BFS level kernel (headline), K8 TC and the conversion
set -x
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bench.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu --no-drivers --no-config5 > $O/r02_ncu_bench.log 2>&1
python tools/ncu_launches.py $O/r02_launches_bench.csv > $O/r02_launches_bench_summary.txt; head -25 $O/r02_launches_bench_summary.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level" -s 4 -c 6 -o $O/r02_ncu_bfs_level \
    python tools/bfs_probe.py --scale 22 --dim 4 --roots 2 > $O/r02_ncu_bfs.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_bfs_level.ncu-rep > $O/r02_ncu_bfs_level.txt; head -60 $O/r02_ncu_bfs_level.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tc_rowhash|k_bmm_masked" -c 2 -o $O/r02_ncu_tc \
    python tools/tc_ab.py 20 4 > $O/r02_ncu_tc.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_tc.ncu-rep > $O/r02_ncu_tc.txt; cat $O/r02_ncu_tc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv|k_rs_|k_tr" -c 12 -o $O/r02_ncu_conv \
    python tools/conv_ab.py 22 4 > $O/r02_ncu_conv.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_conv.ncu-rep > $O/r02_ncu_conv.txt; grep -E "==|time_dur|dram__bytes" $O/r02_ncu_conv.txt
