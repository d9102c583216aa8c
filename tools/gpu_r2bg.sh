set -x
for i in 1 2; do timeout -s KILL 300 python tools/config4.py --scale 24 --no-oracle | python -c "import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print(d['cc'])"; done
