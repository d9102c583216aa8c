set -x
timeout -s KILL 120 python tools/tc_ab.py 20 4,8
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms" 2>&1 | grep -E "Error|assert |passed|failed" | head
timeout -s KILL 300 python -m pytest tests/test_gpu_dist_native.py -q -x -p no:cacheprovider -k "tc or triangle" 2>&1 | tail -1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o gpurun_out/r02_ncu_tcf6 python tools/tc_ab.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_tcf6.ncu-rep | grep -E "==|time_dur|inst_exec|issue_active|warps_active|stalls|dram"
B2SR_PR_MODE=fast timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"k_pr_gather32" -s 3 -c 1 -o gpurun_out/r02_ncu_prf python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_prf.ncu-rep
