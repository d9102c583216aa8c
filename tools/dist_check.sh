# 2 ranks on one GPU over gloo: exercises bench.py's multi-GPU arm end to end
B2SR_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 4 --warmup 3 --scale 20 2>&1 | tail -5
