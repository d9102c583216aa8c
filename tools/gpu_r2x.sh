set -x
O=gpurun_out
timeout -s KILL 120 python tools/h2d_probe.py | tail -1
timeout -s KILL 600 python -m pytest tests/test_gpu_rmat.py tests/test_acceptance_ports.py tests/test_gpu_dist_native.py -q -x -p no:cacheprovider 2>&1 | tail -2
timeout -s KILL 900 python bench.py --no-config5 --no-drivers > $O/r2x_bench.json 2> $O/r2x_bench.err; echo bench rc=$?; tail -3 $O/r2x_bench.err
python -c "import json;d=json.loads(open('$O/r2x_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e']);print({k:(v['transpose_ms'],v['convert_ms']) for k,v in d['sweep'].items()})"
