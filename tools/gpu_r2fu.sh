set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'conversion or rmat or random or roundtrip' 2>&1 | tail -3
timeout -s KILL 600 python -m pytest tests/test_gpu_rmat.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k 'not s26' 2>&1 | tail -3
for r in 1 2; do for v in 0 1; do B2SR_CONV_FUSED=$v timeout -s KILL 300 python tools/conv_ab.py 22 4,8; done; done
for v in 0 1; do B2SR_CONV_FUSED=$v timeout -s KILL 300 python tools/conv_ab.py 24 4; done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_conv|k_scan' --csv --log-file $O/r2fu_launch.csv python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2fu_launch.csv 2>&1 | head -14
