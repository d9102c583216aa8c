timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"bfs|bbb|hot|pull|active|push|update" --csv --log-file gpurun_out/launches_bfs.csv python bench.py --steps 2 --warmup 1 --dims 4 --dim 4 --no-cpu --no-drivers --no-tc > /dev/null 2>&1
python tools/ncu_launches.py gpurun_out/launches_bfs.csv 60 | tail -75
