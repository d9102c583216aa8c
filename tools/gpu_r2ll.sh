set -x
O=gpurun_out
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2ll_launch.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2ll_launch.csv > $O/r2ll_launch.txt 2>&1; head -12 $O/r2ll_launch.txt
