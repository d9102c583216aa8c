set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'transpose or conversion or rmat or random or float_gather' 2>&1 | tail -3
timeout -s KILL 600 python -m pytest tests/test_gpu_rmat.py -q -x -p no:cacheprovider 2>&1 | tail -3
for v in classic onesweep; do B2SR_RS=$v timeout -s KILL 300 python tools/conv_ab.py 22 4,8; done
B2SR_RS=classic timeout -s KILL 300 python tools/conv_ab.py 24 4
timeout -s KILL 300 python tools/conv_ab.py 24 4
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_rs|k_pack4|k_unpack4|k_row_ids' --csv --log-file $O/r2os_launch.csv python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2os_launch.csv 2>&1 | head -20
