set -x
timeout 600 python -m pytest tests/test_acceptance_ports.py -q 2>&1 | tail -15
timeout 900 bash tools/refcheck.sh run 2>&1 | tail -40 > gpurun_out/refcheck.txt; tail -40 gpurun_out/refcheck.txt
timeout 900 python bench.py --workload s26 --steps 16 > gpurun_out/bench_s26.json 2> gpurun_out/bench_s26.err; echo rc=$?
tail -c 3000 gpurun_out/bench_s26.json; tail -20 gpurun_out/bench_s26.err
