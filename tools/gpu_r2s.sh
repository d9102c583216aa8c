set -x
timeout -s KILL 120 python tools/tc_ab.py 20 4,8
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms" 2>&1 | grep -E "Error|assert |passed|failed" | head
B2SR_TRANSPOSE=0 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_tr0.csv python tools/transpose_probe.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r02_launches_tr0.csv | head -30
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o gpurun_out/r02_ncu_tcf5 python tools/tc_ab.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_tcf5.ncu-rep | grep -E "==|time_dur|inst_exec|issue_active|warps_active|stalls"
B2SR_PR_MODE=fast B2SR_PR_TRACE=1 timeout -s KILL 300 python tools/config4.py --scale 24 > gpurun_out/r2s_c4.json 2> gpurun_out/r2s_c4.err; tail -25 gpurun_out/r2s_c4.err
