set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k 'transpose or rmat or random or roundtrip or algorithms or bmm or masked' 2>&1 | tail -3
for r in 1 2; do for v in gather sort; do B2SR_TR8=$v timeout -s KILL 300 python tools/conv_ab.py 22 8; done; done
timeout -s KILL 300 python tools/conv_ab.py 24 8
timeout -s KILL 300 python tools/tc_ab.py 20 4,8
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_rs|k_pack|k_suf|k_scan' --csv --log-file $O/r2t8_launch.csv python tools/conv_ab.py 22 8 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2t8_launch.csv 2>&1 | head -12
