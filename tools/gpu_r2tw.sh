set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k 'transpose or rmat or random or roundtrip or bmv or algorithms' 2>&1 | tail -3
for r in 1 2; do for v in gather sort; do B2SR_TR8=$v timeout -s KILL 300 python tools/conv_ab.py 22 4,16,32; done; done
