set -x
O=gpurun_out
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k "transpose or conversion or rmat_matches or from_coo or roundtrip" 2>&1 | tail -1
timeout -s KILL 200 python tools/conv_ab.py 22 4,8,16
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_tr1.csv python tools/transpose_probe.py > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_tr1.csv | head -14
