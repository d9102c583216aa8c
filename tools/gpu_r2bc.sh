set -x
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "bmv or float_gather or algorithms or golden or config0" 2>&1 | tail -1
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 32 --reps 3 --check
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 16 --reps 3
