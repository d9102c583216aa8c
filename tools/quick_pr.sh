timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "float_gather or algorithms or rmat or random" 2>&1 | tail -2
timeout 900 python tools/config4.py --scale 24 2>&1 | tail -1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bff|pr_|pw_|relax|cc_|vlong" -c 60 --csv --log-file gpurun_out/launches_pr.csv python tools/config4.py --scale 24 --no-oracle > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_pr.csv | head -16
