cd $GRAFT_REPO_ROOT
MPSG_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config c2 --steps 2 --warmup 3 --e2e-steps 1 2>&1 | grep -v Warning | tail -3
MPSG_BENCH_SHARE_DEVICE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config c2 --impl reference --steps 1 --warmup 1 2>&1 | grep -v Warning | tail -2
