set -x
timeout -s KILL 120 python tools/tc_ab.py 20 4,8
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "bmm or masked_spgemm or algorithms or transpose" 2>&1 | grep -E "Error|assert |passed|failed" | head
for v in 0 1 2 3; do echo prg=$v; B2SR_PRG=$v B2SR_PR_MODE=fast B2SR_PR_TRACE=1 timeout -s KILL 200 python tools/config4.py --scale 24 --no-oracle 2>&1 >/dev/null | grep "sweep [5-9]" | head -3; done
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_bmv_bbb_stream" -s 2 -c 1 -o gpurun_out/r02_ncu_k4 python tools/spmv_probe.py --dims 4 --reps 3 > /dev/null 2>&1
python tools/ncu_kv.py gpurun_out/r02_ncu_k4.ncu-rep
