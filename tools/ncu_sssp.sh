timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bff|vlong|relax|cc_" -c 400 --csv --log-file gpurun_out/launches_sssp.csv python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_sssp.csv | head -20
