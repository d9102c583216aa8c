set -x
timeout 300 python tools/h2d_probe.py > gpurun_out/h2d.json 2> gpurun_out/h2d.err; cat gpurun_out/h2d.json; tail -3 gpurun_out/h2d.err
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
