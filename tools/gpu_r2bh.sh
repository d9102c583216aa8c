set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2bh_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/r2bh_pytest.log
timeout -s KILL 900 python bench.py > $O/r2bh_bench.json 2> $O/r2bh_bench.err; echo bench rc=$?; tail -2 $O/r2bh_bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2bh_ref.json 2> $O/r2bh_ref.err; echo ref rc=$?
