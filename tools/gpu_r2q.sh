set -x
timeout -s KILL 120 python tools/tc_ab.py 20 4,8
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms" 2>&1 | grep -E "Error|assert |passed|failed" | head
B2SR_TC_SYM=0 timeout -s KILL 120 python tools/tc_ab.py 20 4
for b in 4096 32000; do B2SR_TC_BUDGET=$b timeout -s KILL 120 python tools/tc_ab.py 20 4; done
timeout -s KILL 300 python -m pytest tests/test_gpu_dist_native.py -q -x -p no:cacheprovider -k "tc or triangle" 2>&1 | tail -1
timeout -s KILL 300 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "triangle" 2>&1 | tail -1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o gpurun_out/r02_ncu_tcf4 python tools/tc_ab.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_tcf4.ncu-rep
