set -x
O=gpurun_out
B2SR_PR_TRACE=1 timeout -s KILL 300 python tools/config4.py --scale 24 --no-oracle 2>&1 >/dev/null | grep "sweep [3-5]" | head -6
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_pr_exact.csv python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_pr_exact.csv | head -30
