#!/bin/bash
# compute-sanitizer over the golden-fixture parity tests (every entry point on
# small inputs): memcheck (out-of-bounds / misaligned accesses, including the
# 32-bit red.or stores on padded bit vectors), racecheck (shared-memory
# hazards: hot-column cache staging, TC row staging and hit queues, merge
# buffers, block scans) and synccheck (barrier / warp-sync misuse).
# Logs -> gpurun_out/san_*.{log,pytest}.
set -x
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_parity.py tests/test_acceptance_ports.py"
K="not rmat_against and not concurrent and not float_gather_long and not hot_column"
timeout -s KILL 1500 $CS --tool memcheck --leak-check no --print-limit 50 --log-file $O/san_memcheck.log \
    python -m pytest $SEL tests/test_gpu_dist_native.py -q -x -p no:cacheprovider -k "$K and not two_ranks and not thread_ranks" > $O/san_memcheck.pytest 2>&1
echo memcheck rc=$?; tail -3 $O/san_memcheck.pytest; tail -5 $O/san_memcheck.log
timeout -s KILL 1200 $CS --tool racecheck --racecheck-report hazard --print-limit 50 --log-file $O/san_racecheck.log \
    python -m pytest $SEL -q -x -p no:cacheprovider -k "$K" > $O/san_racecheck.pytest 2>&1
echo racecheck rc=$?; tail -3 $O/san_racecheck.pytest; tail -5 $O/san_racecheck.log
timeout -s KILL 900 $CS --tool synccheck --print-limit 50 --log-file $O/san_synccheck.log \
    python -m pytest $SEL -q -x -p no:cacheprovider -k "$K" > $O/san_synccheck.pytest 2>&1
echo synccheck rc=$?; tail -3 $O/san_synccheck.pytest; tail -5 $O/san_synccheck.log
