# TC filter kernel v2 (hit queue, shuffle row search) + warp-merge conversion: parity, timing, ncu
set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "conversion or bmm or masked_spgemm or algorithms or worked" 2>&1 | grep -E "Error|assert|passed|failed" | head -20
timeout 300 python tools/tc_ab.py 20 4,8
for b in 4096 32000; do B2SR_TC_BUDGET=$b timeout 300 python tools/tc_ab.py 20 4; done
timeout 300 python tools/conv_ab.py 22 4,8; B2SR_CONV_MERGE=0 timeout 300 python tools/conv_ab.py 22 4,8
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter|k_conv_merge" -c 3 -o $O/r02_ncu_tcf2 \
    python tools/tc_ab.py 20 4 > $O/r02_ncu_tcf2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_conv" -c 4 -o $O/r02_ncu_conv2 \
    python tools/conv_ab.py 22 4 > $O/r02_ncu_conv2.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_tcf2.ncu-rep > $O/r02_ncu_tcf2.txt; cat $O/r02_ncu_tcf2.txt
python tools/ncu_kv.py $O/r02_ncu_conv2.ncu-rep > $O/r02_ncu_conv2.txt; cat $O/r02_ncu_conv2.txt
