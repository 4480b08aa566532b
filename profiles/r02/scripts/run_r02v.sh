# multi-rank bench path end to end with two ranks sharing the one GPU (gloo; NCCL refuses a
# duplicated device): barriers, max-over-ranks timing, pair offsets, P_global, rank-0 line
export ODPO_SHARE_GPU=1 ODPO_DIST_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --config pythia --steps 5 --warmup 3 --no-aux --no-e2e 2>/dev/null | tail -1 | cut -c1-600
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 2>/dev/null | tail -1 | cut -c1-300
