set -x
O=gpurun_out
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 32 --reps 3
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_bff16.csv python tools/bff_probe.py --scale 16 --dim 32 --reps 2 > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_bff16.csv 40
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:"bff|vlong" -s 0 -c 6 -o $O/r02_ncu_bff16 python tools/bff_probe.py --scale 16 --dim 32 --reps 1 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_bff16.ncu-rep
