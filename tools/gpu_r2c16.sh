set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'conversion or rmat or random or roundtrip' 2>&1 | tail -3
for r in 1 2; do for v in 0 1; do B2SR_CONV_FUSED=$v timeout -s KILL 300 python tools/conv_ab.py 22 4,16; done; done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2c16_launch.csv python tools/conv_ab.py 22 16 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2c16_launch.csv 2>&1 | head -16
