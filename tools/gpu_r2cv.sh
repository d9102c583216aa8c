set -x
O=gpurun_out
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2cv_launch.csv python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2cv_launch.csv 2>&1 | head -30
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_conv_count_hash -c 1 -o $O/r02_ncu_convhash python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_convhash.ncu-rep
