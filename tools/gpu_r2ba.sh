set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k "transpose or rmat_matches or from_coo or roundtrip or conversion or algorithms" 2>&1 | tail -1
for i in 1 2; do timeout -s KILL 200 python tools/conv_ab.py 22 4,8; done
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_tr3.csv python tools/transpose_probe.py > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/r02_launches_tr3.csv 2>/dev/null | head -8
