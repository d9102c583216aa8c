set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmv or float_gather or algorithms or golden or worked" 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "config0" 2>&1 | tail -1
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 32 --reps 3 --check
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 16 --reps 3
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bffcsr.csv python tools/bff_probe.py --scale 16 --dim 32 --reps 2 > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r02_launches_bffcsr.csv 2>/dev/null | head -8
