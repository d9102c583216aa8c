set -x
O=gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmv or float_gather or algorithms or golden or worked" 2>&1 | tail -1
timeout -s KILL 900 python -m pytest tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "config0" 2>&1 | tail -1
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 32 --reps 3 --check
timeout -s KILL 120 python tools/bff_probe.py --scale 16 --dim 16 --reps 3 --check
timeout -s KILL 600 python bench.py --no-config5 --no-drivers --no-tc --no-cpu --dims 4,8 > $O/r2ae_bench.json 2> $O/r2ae_bench.err; echo rc=$?
python -c "import json;d=json.loads(open('$O/r2ae_bench.json').read().strip().splitlines()[-1]);print(d['value'],d['roofline']['kernel_ms'],d['roofline']['frac'],d['e2e']['value'],d['e2e']['breakdown_ms']);print({k:(v['spmv_ms'],v['spmv_frac'],v['bfs_gteps']) for k,v in d['sweep'].items()})"
