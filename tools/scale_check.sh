#!/bin/bash
# Weak scaling of the default workload at 2..NGPU GPUs with the current build (bench.py under torchrun, NCCL).
# Usage (under gpurun --gpus N): NGPU=4 bash tools/scale_check.sh <tag>
tag=${1:-rX}
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/${tag}_scale_build.log 2>&1
n=2
while [ $n -le ${NGPU:-2} ]; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29600 + n)) bench.py --gpus $n > $out/${tag}_scale${n}.json 2> $out/${tag}_scale${n}.err
  echo "scale${n}=$?" >> $out/${tag}_scale_status.txt
  n=$((n * 2))
done
cat $out/${tag}_scale_status.txt
