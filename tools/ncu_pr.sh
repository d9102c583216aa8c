timeout 900 python tools/config4.py --scale 24 --no-oracle 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bff|pr_|pw_|relax|cc_|vlong" -c 200 --csv --log-file gpurun_out/launches_pr.csv python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_pr.csv 30
