# round-2 re-entry check: all GPU tests, smoke, the default bench, launch list
set -x
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2m_pytest.log 2>&1; echo pytest rc=$?; tail -3 $O/r2m_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py > $O/r2m_bench.json 2> $O/r2m_bench.err; echo bench rc=$?; tail -c 600 $O/r2m_bench.json; tail -3 $O/r2m_bench.err
