set -x
for i in 1 2 3; do timeout -s KILL 300 python tools/tc_ab.py 20 4; done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o gpurun_out/r02_ncu_tc7 python tools/tc_ab.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_tc7.ncu-rep | grep -E "==|time_dur|inst_exec|issue_active|warps_active|stalls"
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv
