set -x
O=gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_acceptance_ports.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "config0 or config1_s16 or s16" 2>&1 | tail -2
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 32 --reps 3 --check
B2SR_BFF_CSR=0 timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 32 --reps 3
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 16 --reps 3
timeout -s KILL 120 python tools/spmv_probe.py --dims 4,8 --reps 5
