set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_rmat.py tests/test_acceptance_ports.py tests/test_gpu_dist_native.py -q -x -p no:cacheprovider -k "large_host or container or from_blocks or e2e or block" 2>&1 | tail -1
for p in 1 0; do B2SR_H2D_PACK=$p timeout -s KILL 120 python tools/upload_probe.py | tail -1; done
timeout -s KILL 600 python bench.py --no-config5 --no-drivers --no-tc --no-cpu --dims 4 > $O/r2as_b.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/r2as_b.json').read().strip().splitlines()[-1]);print(d['value'],d['e2e'])"
