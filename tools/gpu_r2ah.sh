set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2ah_pytest.log 2>&1; echo pytest rc=$?; tail -3 $O/r2ah_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 900 python bench.py > $O/r2ah_bench.json 2> $O/r2ah_bench.err; echo bench rc=$?; tail -3 $O/r2ah_bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2ah_ref.json 2> $O/r2ah_ref.err; echo ref rc=$?; tail -c 800 $O/r2ah_ref.json
