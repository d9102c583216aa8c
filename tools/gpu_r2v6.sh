set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2v6_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/r2v6_pytest.log
timeout -s KILL 900 python bench.py > $O/r2v6_bench.json 2> $O/r2v6_bench.err; echo bench rc=$?; tail -2 $O/r2v6_bench.err
timeout -s KILL 1500 python bench.py --workload s26 > $O/r2v6_s26.json 2> $O/r2v6_s26.err; echo s26 rc=$?; tail -2 $O/r2v6_s26.err
timeout -s KILL 300 python tools/upload_probe.py 22 > $O/r2v6_upload.json
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:'k_conv_compact|k_pack4_rows|k_rs_scatter' -c 6 -o $O/r02_ncu_convtr2 python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_convtr2.ncu-rep > $O/r2v6_ncu_convtr2.txt 2>&1
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2v6_convtr_launch.csv python tools/conv_ab.py 22 4 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2v6_convtr_launch.csv > $O/r2v6_convtr_launch.txt 2>&1
