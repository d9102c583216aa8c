set -x
O=gpurun_out
timeout -s KILL 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/r2v7_pytest.log 2>&1; echo pytest rc=$?; tail -2 $O/r2v7_pytest.log
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout -s KILL 900 python bench.py > $O/r2v7_bench.json 2> $O/r2v7_bench.err; echo bench rc=$?; tail -2 $O/r2v7_bench.err
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/r2v7_ref.json 2> $O/r2v7_ref.err; echo ref rc=$?
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r2v7_launch.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
python tools/ncu_launches.py $O/r2v7_launch.csv > $O/r2v7_launch.txt 2>&1; head -30 $O/r2v7_launch.txt
