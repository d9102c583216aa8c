#!/bin/bash
# compute-sanitizer over the golden-fixture parity tests (every entry point on
# small inputs): memcheck (out-of-bounds / misaligned accesses, including the
# 32-bit red.or stores on padded bit vectors), racecheck (shared-memory
# hazards: hot-column cache staging, row-hash tables, block scans) and
# synccheck (barrier / warp-sync misuse).  Logs -> gpurun_out/san_*.log.
set -x
O=gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tests/test_gpu_parity.py tests/test_acceptance_ports.py"
timeout 2400 $CS --tool memcheck --leak-check no --print-limit 50 --log-file $O/san_memcheck.log \
    python -m pytest $SEL tests/test_gpu_dist_native.py -q -x -p no:cacheprovider -k "not two_ranks and not thread_ranks[3" > $O/san_memcheck.pytest 2>&1
echo memcheck rc=$?; tail -3 $O/san_memcheck.pytest; tail -5 $O/san_memcheck.log
timeout 2400 $CS --tool racecheck --racecheck-report hazard --print-limit 50 --log-file $O/san_racecheck.log \
    python -m pytest $SEL -q -x -p no:cacheprovider > $O/san_racecheck.pytest 2>&1
echo racecheck rc=$?; tail -3 $O/san_racecheck.pytest; tail -5 $O/san_racecheck.log
timeout 2400 $CS --tool synccheck --print-limit 50 --log-file $O/san_synccheck.log \
    python -m pytest $SEL -q -x -p no:cacheprovider > $O/san_synccheck.pytest 2>&1
echo synccheck rc=$?; tail -3 $O/san_synccheck.pytest; tail -5 $O/san_synccheck.log
