# one GPU call: parity tests, config-4 drivers at s24, x-gather A/B, BFS trace + launch list
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/config4.py --scale 24 > gpurun_out/config4_s24.json 2> gpurun_out/config4.err; echo c4=$?
cat gpurun_out/config4_s24.json; tail -2 gpurun_out/config4.err
bash tools/ab_xgather.sh
