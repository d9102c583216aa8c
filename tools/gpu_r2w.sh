set -x
O=gpurun_out
timeout -s KILL 120 python tools/h2d_probe.py
for t in 8 16; do B2SR_H2D_THREADS=$t timeout -s KILL 120 python tools/h2d_probe.py | tail -1; done
timeout -s KILL 60 tools/bin/micro_bmma; timeout -s KILL 60 tools/bin/micro_popc
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2w_pytest.log 2>&1; echo pytest rc=$?; tail -3 $O/r2w_pytest.log
timeout -s KILL 900 python bench.py > $O/r2w_bench.json 2> $O/r2w_bench.err; echo bench rc=$?; tail -3 $O/r2w_bench.err
