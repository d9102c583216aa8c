# round-2 ncu evidence (profiles/r02_*): launch list of a short default bench,
# full captures of the headline BFS level kernel, K4, K8 TC, the K1/K2 warp
# merge and the fast PageRank gather (one launch each), summarised to text.
set -x
O=gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bench.csv \
    python bench.py --steps 4 --warmup 3 --no-cpu --no-drivers --no-config5 > $O/r02_ncu_bench.log 2>&1
python tools/ncu_launches.py $O/r02_launches_bench.csv > $O/r02_launches_bench_summary.txt; head -30 $O/r02_launches_bench_summary.txt
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_bfs_level" -s 8 -c 3 -o $O/r02_ncu_bfs_level \
    python tools/bfs_probe.py --scale 22 --dim 4 --roots 3 > $O/r02_ncu_bfs.log 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_bmv_bbb_stream" -s 2 -c 1 -o $O/r02_ncu_k4 \
    python tools/spmv_probe.py --dims 4 --reps 3 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o $O/r02_ncu_tc \
    python tools/tc_ab.py 20 4 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_conv_merge" -c 2 -o $O/r02_ncu_conv \
    python tools/conv_ab.py 22 4 > /dev/null 2>&1
B2SR_PR_MODE=fast timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_pr_gather32" -s 3 -c 1 \
    -o $O/r02_ncu_prfast python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
for r in bfs_level k4 tc conv prfast; do python tools/ncu_kv.py $O/r02_ncu_$r.ncu-rep > $O/r02_ncu_$r.txt; done
cat $O/r02_ncu_bfs_level.txt | head -40
