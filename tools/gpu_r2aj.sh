set -x
O=gpurun_out
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_tc26.csv -k regex:"k_tc_filter|k_bmm_masked_items|k_tcf|k_tc_item" python tools/tc_ab.py 26 4 > $O/r2aj_tc26.log 2>&1
python tools/ncu_launches.py $O/r02_launches_tc26.csv | head -12; tail -2 $O/r2aj_tc26.log
