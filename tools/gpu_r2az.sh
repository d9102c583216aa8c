set -x
O=gpurun_out
free -g | head -2; nproc
( time timeout -s KILL 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > $O/r2az_ref26.json 2> $O/r2az_ref26.err ) 2>&1 | tail -3
echo rc=$?; tail -c 1500 $O/r2az_ref26.json; tail -3 $O/r2az_ref26.err
