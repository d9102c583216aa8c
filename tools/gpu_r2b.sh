set -x
timeout 900 python -m pytest tests/test_gpu_dist_native.py -x -q 2>&1 | tail -30
for t in 8 12 16; do B2SR_H2D_THREADS=$t timeout 300 python tools/h2d_probe.py; done
