# Exercise bench.py's multi-rank path (barrier, max-over-ranks timing,
# summed counts, rank-0 printing) on a ONE-GPU box: both ranks share cuda:0
# and use gloo collectives (BODE_BENCH_SHARED_GPU=1).  Timing is meaningless
# here; the driver's real N-GPU runs use one GPU per rank and NCCL.
BODE_BENCH_SHARED_GPU=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu
BODE_BENCH_SHARED_GPU=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --scaling weak --no-cpu --no-e2e
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29512 bench.py --impl reference --gpus 2 --steps 1 --warmup 1
