set -x
O=gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_rmat.py -q -x -p no:cacheprovider -k "bfs or algorithms or hot_column or sssp or rmat_against" 2>&1 | tail -1
for i in 1 2; do timeout -s KILL 600 python bench.py --no-config5 --no-drivers --no-tc --no-cpu --dims 4 > $O/r2ar_b$i.json 2>/dev/null; python -c "import json;d=json.loads(open('$O/r2ar_b$i.json').read().strip().splitlines()[-1]);print(d['value'],d['ms_per_step'],d['roofline']['kernel_ms'],d['sweep']['4']['bfs_gteps'])"; done
