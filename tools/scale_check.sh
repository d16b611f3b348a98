#!/bin/bash
# Multi-GPU check of the bench contract (under gpurun --gpus N): the default command with --gpus N re-executes itself
# under torchrun; the reference arm under torchrun prints from rank 0 only.  Usage: bash tools/scale_check.sh N TAG
n=${1:-2}; tag=${2:-s$n}
mkdir -p gpurun_out
timeout 1200 python bench.py --gpus $n > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench=$?"
grep -c "NCCL INFO" gpurun_out/${tag}_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus $n --impl reference --steps 1 --warmup 0 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err
echo "ref=$?"
