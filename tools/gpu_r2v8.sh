set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2v8_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/r2v8_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -s KILL 900 python bench.py > $O/r2v8_bench.json 2> $O/r2v8_bench.err; echo bench rc=$?; tail -2 $O/r2v8_bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2v8_ref.json 2> $O/r2v8_ref.err; echo ref rc=$?
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_bfs_update_dc -c 3 -o $O/r02_ncu_bfsupd python tools/bfs_time.py 20 4 > /dev/null 2>&1
python tools/ncu_kv.py $O/r02_ncu_bfsupd.ncu-rep > $O/r2v8_ncu_bfsupd.txt 2>&1
