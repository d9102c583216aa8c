# round-2 final captures of the kernels changed after tools/profile_r2.sh
set -x
O=gpurun_out
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_conv_count_hash|k_conv_merge|k_rs_scatter|k_rs_hist|k_unpack4" -s 20 -c 8 -o $O/r02_ncu_convtr python tools/conv_ab.py 22 4 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_bff_csr" -s 2 -c 2 -o $O/r02_ncu_bffcsr python tools/bff_probe.py --scale 16 --dim 32 --reps 2 > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:"k_tc_filter" -c 1 -o $O/r02_ncu_tcfinal python tools/tc_ab.py 20 4 > /dev/null 2>&1
for r in convtr bffcsr tcfinal; do python tools/ncu_kv.py $O/r02_ncu_$r.ncu-rep > $O/r02_ncu_$r.txt; done
grep -E "==|time_dur|dram__bytes|inst_exec|issue_active" $O/r02_ncu_convtr.txt $O/r02_ncu_bffcsr.txt $O/r02_ncu_tcfinal.txt
