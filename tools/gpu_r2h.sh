set -x
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_dist_native.py -q -x 2>&1 | tail -5
for p in 0 1; do B2SR_PR_L2PERSIST=$p B2SR_PR_TRACE=1 B2SR_PR_MODE=fast timeout 600 python tools/config4.py --scale 24 --no-oracle 2>&1 | grep -E "sweep [0-2] |pagerank" | cut -c1-300; done
B2SR_PR_MODE=fast timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pr_gather32" -s 2 -c 1 -o $O/r02_ncu_pr_fast python tools/config4.py --scale 24 --no-oracle > $O/r02_ncu_pr.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_pr_fast.ncu-rep > $O/r02_ncu_pr_fast.txt; cat $O/r02_ncu_pr_fast.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_conv$" -c 2 -o $O/r02_ncu_conv python tools/conv_ab.py 22 4 > $O/r02_ncu_conv.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_conv.ncu-rep > $O/r02_ncu_conv.txt; cat $O/r02_ncu_conv.txt
