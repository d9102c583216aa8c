timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for V in "B2SR_STREAM_THREADS=768" "B2SR_STREAM_THREADS=1024"; do echo $V; env $V timeout 300 python tools/spmv_probe.py --reps 8 --dims 4; done
