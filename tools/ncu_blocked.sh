# ncu full captures of the blocked and row-major bbb kernels at s22 d=4
timeout 500 ncu --set full --clock-control none --import-source on -k regex:"k_blocked|k_bmv_bbb" -s 2 -c 2 -o gpurun_out/prof_blk python bench.py --steps 1 --warmup 1 --dims 4 --dim 4 --no-tc --no-cpu > gpurun_out/ncu_blk.out 2>&1
echo ncu=$?
B2SR_BLOCKED=0 timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_bmv_bbb" -s 2 -c 1 -o gpurun_out/prof_rm python bench.py --steps 1 --warmup 1 --dims 4 --dim 4 --no-tc --no-cpu > gpurun_out/ncu_rm.out 2>&1
echo ncu=$?
