set -x
timeout 600 python tools/conv_ab.py 22
timeout 900 python -m pytest tests/test_gpu_configs.py -q -x 2>&1 | tail -5
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
tail -c 4000 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
