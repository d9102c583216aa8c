# TC row-filter kernel: parity of the K8 paths, s20 timing vs the items kernel, ncu of the new kernel
set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms or worked or rmat_against" 2>&1 | tail -3
timeout 300 python tools/tc_ab.py 20 4,8; B2SR_TC_FILTER=0 timeout 300 python tools/tc_ab.py 20 4,8
for b in 4096 8192 32000; do B2SR_TC_BUDGET=$b timeout 300 python tools/tc_ab.py 20 4; done
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "triangle" 2>&1 | tail -3
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o $O/r02_ncu_tcf \
    python tools/tc_ab.py 20 4 > $O/r02_ncu_tcf.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_tcf.ncu-rep > $O/r02_ncu_tcf.txt; head -80 $O/r02_ncu_tcf.txt
