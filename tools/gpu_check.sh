# parity tests, smoke, default bench
set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
