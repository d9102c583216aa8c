set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_acceptance_ports.py -q -k "bmm or tc or triangle or config2 or config1 or criterion" 2>&1 | tail -5
for h in 0 1; do B2SR_TC_HASH=$h timeout 300 python tools/tc_ab.py 20 4,8; done
B2SR_TC_HASH=1 timeout 600 python tools/tc_ab.py 24 4
timeout 600 python tools/conv_ab.py 22
