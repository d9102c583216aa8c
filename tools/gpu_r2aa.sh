set -x
O=gpurun_out
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "transpose or conversion or algorithms or roundtrip" 2>&1 | tail -1
timeout -s KILL 200 python tools/conv_ab.py 22 4,8
bash tools/profile_r2.sh
timeout -s KILL 900 python bench.py > $O/r2aa_bench.json 2> $O/r2aa_bench.err; echo bench rc=$?; tail -3 $O/r2aa_bench.err
