set -x
for v in 1 all; do echo csr=$v; B2SR_BFF_CSR=$v B2SR_PR_TRACE=1 timeout -s KILL 300 python tools/config4.py --scale 24 --no-oracle 2>&1 >/dev/null | grep "sweep [4-6]" | head -3; done
B2SR_BFF_CSR=all timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmv or float_gather or algorithms or golden" 2>&1 | tail -1
