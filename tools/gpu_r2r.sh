set -x
timeout -s KILL 120 python tools/tc_ab.py 20 4,8
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms or transpose or conversion" 2>&1 | grep -E "Error|assert |passed|failed" | head
timeout -s KILL 200 python tools/conv_ab.py 22 4,8
B2SR_TRANSPOSE=0 timeout -s KILL 200 python tools/conv_ab.py 22 4
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"k_tr_|k_tc_filter" -c 4 -o gpurun_out/r02_ncu_tr1 python tools/tc_ab.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_tr1.ncu-rep | grep -E "==|time_dur|dram__bytes|inst_exec|issue_active|stalls"
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_conv.csv python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r02_launches_conv.csv | head -30
