set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'transpose or rmat or random or roundtrip' 2>&1 | tail -3
timeout -s KILL 600 python tools/conv_ab.py 22 4,8,16,32
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_transpose_gather' --csv --log-file $O/r2tg_launch.csv python tools/conv_ab.py 22 8 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2tg_launch.csv 2>&1 | head -5
