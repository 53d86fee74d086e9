# usage (under gpurun): bash tools/gpu/torchrun_n1.sh -> bench.py launched by torchrun on the one GPU
# (NCCL process group of size 1: the multi-rank code path, counter all_reduce and max-over-ranks timing)
mkdir -p gpurun_out
NCCL_DEBUG=INFO timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-cufft \
  > gpurun_out/torchrun_n1.log 2> gpurun_out/torchrun_n1.err; echo "torchrun rc=$?" >> gpurun_out/torchrun_n1.err
NCCL_DEBUG=WARN timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29534 bench.py --gpus 1 --steps 2 --warmup 3 --scaling strong --no-e2e --no-cpu-baseline --no-cufft \
  > gpurun_out/torchrun_n1_strong.log 2>&1; echo "strong rc=$?" >> gpurun_out/torchrun_n1_strong.log
