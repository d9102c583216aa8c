set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k 'transpose or rmat or random or roundtrip or coo or conversion' 2>&1 | tail -3
for r in 1 2; do timeout -s KILL 300 python tools/conv_ab.py 22 4,8; done
timeout -s KILL 300 python tools/conv_ab.py 24 4
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_rs|k_transpose|k_trp|k_row|k_iota|k_pack|k_unpack|k_scan' --csv --log-file $O/r2rk_launch.csv python tools/conv_ab.py 22 8 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2rk_launch.csv 2>&1 | head -14
