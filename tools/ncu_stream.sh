timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_bmv_bbb_stream|k_hot_fill|k_and_words" -s 6 -c 6 -o gpurun_out/ncu_stream python tools/spmv_probe.py --reps 3 > gpurun_out/ncu_stream.log 2>&1; tail -2 gpurun_out/ncu_stream.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_spmv.csv python tools/spmv_probe.py --reps 3 > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_spmv.csv 40
