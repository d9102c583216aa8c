set -x
O=gpurun_out
timeout -s KILL 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --workload s26 --steps 4 --warmup 3 --no-cpu > $O/r2av_s26.json 2> $O/r2av_s26.err; echo rc=$?
tail -c 2500 $O/r2av_s26.json; tail -5 $O/r2av_s26.err
