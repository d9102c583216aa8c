set -x
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -q -x -p no:cacheprovider -k "algorithms or golden or config3 or random_sweep" 2>&1 | tail -1
B2SR_PR_TRACE=0 timeout -s KILL 300 python tools/config4.py --scale 24 --no-oracle | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print({k:v for k,v in d.items() if k in ('cc','sssp','pagerank')})"
