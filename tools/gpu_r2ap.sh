set -x
timeout -s KILL 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter<4, true, true>|k_tc_filter" --launch-skip 1 -c 1 -o gpurun_out/r02_ncu_tcr26 python tools/tc_ab.py 26 4 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_tcr26.ncu-rep | grep -E "==|time_dur|inst_exec|issue_active|warps_active|stalls"
