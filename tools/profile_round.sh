# ncu evidence for profiles/: full capture of the K4 stream kernel (d=4, 8) at s22,
# its per-launch DRAM traffic, and the launch list of one short bench run
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bmv_bbb_stream" -s 2 -c 2 -o gpurun_out/ncu_k4 python tools/spmv_probe.py --reps 3 --dims 4,8 > gpurun_out/ncu_k4.log 2>&1
python tools/traffic_json.py gpurun_out/ncu_k4.ncu-rep 22 gpurun_out/traffic.json
python tools/ncu_kv.py gpurun_out/ncu_k4.ncu-rep > gpurun_out/ncu_k4_summary.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 4 --warmup 3 --dims 4 --dim 4 --no-cpu --no-drivers --no-tc > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_bench.csv > gpurun_out/launches_bench_summary.txt
head -30 gpurun_out/launches_bench_summary.txt
