#!/bin/bash
# Every BASELINE.json config at N=1 through bench.py (the fused-kernel path only: no CPU baseline, no f2 extras), and,
# with NGPU > 1, the Qwen3-32B-shaped strong-scaling points at 2..NGPU GPUs.
# Usage (under gpurun): [NGPU=4] bash tools/config_sweep.sh <tag>
tag=${1:-rX}
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/${tag}_sweep_build.log 2>&1
for c in qwen3-4b qwen2.5-7b qwen3-30b-a3b qwen3-32b; do
  timeout 900 python bench.py --config $c --no-cpu-baseline --no-f2 --no-f2-train \
      > $out/${tag}_cfg_${c}.json 2> $out/${tag}_cfg_${c}.err; echo "cfg_${c}=$?" >> $out/${tag}_sweep_status.txt
done
n=2
while [ $n -le ${NGPU:-1} ]; do
  for c in qwen3-32b; do
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
        --master-port $((29500 + n)) bench.py --gpus $n --config $c --scaling strong --no-cpu-baseline --no-f2 \
        --no-f2-train > $out/${tag}_strong${n}_${c}.json 2> $out/${tag}_strong${n}_${c}.err
    echo "strong${n}_${c}=$?" >> $out/${tag}_sweep_status.txt
  done
  n=$((n * 2))
done
cat $out/${tag}_sweep_status.txt
# the default bench line (with the CPU-oracle baseline); compute-sanitizer is closed on this GPU pool
timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench=$?" >> $out/${tag}_sweep_status.txt
cat $out/${tag}_sweep_status.txt
