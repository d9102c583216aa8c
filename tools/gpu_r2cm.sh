set -x
O=gpurun_out
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_conv_merge -c 1 -o $O/r02_ncu_convmerge python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_convmerge.ncu-rep
