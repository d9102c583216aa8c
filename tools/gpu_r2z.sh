set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py tests/test_acceptance_ports.py -q -x -p no:cacheprovider 2>&1 | tail -1
timeout -s KILL 200 python tools/conv_ab.py 22 4,8,16,32
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02_launches_tr2.csv python tools/transpose_probe.py > /dev/null 2>&1
python tools/ncu_launches.py $O/r02_launches_tr2.csv > $O/r02_launches_tr2.txt; head -14 $O/r02_launches_tr2.txt
