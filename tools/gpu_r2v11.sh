set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2v11_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/r2v11_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -s KILL 900 python bench.py > $O/r2v11_bench.json 2> $O/r2v11_bench.err; echo bench rc=$?; tail -2 $O/r2v11_bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2v11_ref.json 2> $O/r2v11_ref.err; echo ref rc=$?
timeout -s KILL 1500 python bench.py --workload s26 > $O/r2v11_s26.json 2> $O/r2v11_s26.err; echo s26 rc=$?
