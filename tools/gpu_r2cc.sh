set -x
O=gpurun_out
for r in 1 2; do for v in rowid rows; do B2SR_TR_PACK=$v timeout -s KILL 300 python tools/conv_ab.py 22 4; done; done
timeout -s KILL 300 python tools/cc_probe.py 24
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2cc_launch.csv python tools/cc_probe.py 24 1 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2cc_launch.csv 2>&1 | head -24
