set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms" 2>&1 | tail -2
timeout 300 python tools/tc_ab.py 20 4,8
timeout 300 python tools/h2d_probe.py
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o $O/r02_ncu_tcf3 python tools/tc_ab.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_tcf3.ncu-rep
