set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_dist_native.py tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "tc or triangle or masked_spgemm or bmm" 2>&1 | tail -1
timeout -s KILL 900 python tools/config5.py --roots 2 > $O/r2ai_c5.json 2> $O/r2ai_c5.err; echo c5 rc=$?; cat $O/r2ai_c5.json | head -c 1500; tail -2 $O/r2ai_c5.err
timeout -s KILL 900 python bench.py --no-tc --no-drivers --no-cpu --dims 4 --steps 8 > $O/r2ai_bench.json 2> $O/r2ai_bench.err; echo bench rc=$?
python -c "import json;d=json.loads(open('$O/r2ai_bench.json').read().strip().splitlines()[-1]);c=d['config5_n1'];print(c['bfs_gteps'],c['tc'],d['clocks'])"
