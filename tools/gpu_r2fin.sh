set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2fin_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/r2fin_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -s KILL 900 python bench.py > $O/r2fin_bench.json 2> $O/r2fin_bench.err; echo bench rc=$?
