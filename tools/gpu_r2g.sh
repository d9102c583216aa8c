set -x
O=gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_conv.csv python tools/conv_ab.py 22 > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_conv.csv | head -30
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv<" -c 8 -o $O/r02_ncu_conv python tools/conv_ab.py 22 4,32 > $O/r02_ncu_conv.log 2>&1
python tools/ncu_kv.py $O/r02_ncu_conv.ncu-rep > $O/r02_ncu_conv.txt; cat $O/r02_ncu_conv.txt
B2SR_PR_TRACE=1 B2SR_PR_MODE=fast timeout 600 python tools/config4.py --scale 24 --no-oracle 2>&1 | tail -25
