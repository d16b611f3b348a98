#!/bin/bash
# One GPU-box session: smoke, the GPU parity suite, the default bench (and its reference arm), the ncu launch list
# of the bench and one ncu --set full capture per kernel family.  Usage (under gpurun): bash tools/gpu_round.sh <tag>
# Env (set inside the gpurun command): PYTEST=0 / BENCH=0 / NCU=0 skip those parts.
tag=${1:-rX}
out=gpurun_out
mkdir -p $out
st=$out/${tag}_status.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $out/${tag}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo "smoke=$?" >> $st
if [ "${PYTEST:-1}" = "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -s --timeout 600 --timeout_method thread -rf > $out/${tag}_pytest.log 2>&1
  echo "pytest=$?" >> $st
fi
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench=$?" >> $st
  timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err
  echo "bench_ref=$?" >> $st
fi
if [ "${NCU:-1}" = "1" ]; then
  # launch list of the bench command (one timed step after one warm-up: 32B batch = 256 micro-batches per step)
  timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/${tag}_ncu_plain.log 2>&1 && \
  timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
      python bench.py --steps 1 --warmup 1 --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1; echo "ncu_launches=$?" >> $st
  # the fused (3)-(5) kernel (AUTO = oct tile) on one 32768-row micro-batch of the bench's workload
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:policy_loss_quad -s 1 -c 1 -o $out/${tag}_kernel \
      python tools/prof_kernel.py --config qwen3-32b --algos oct_reg --reps 1 --warmup 1 > $out/${tag}_ncu_full.log 2>&1
  echo "ncu_full=$?" >> $st
  # f1: the one-warp-per-row log-prob kernel
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:token_logp_warp -s 1 -c 1 -o $out/${tag}_f1 \
      python tools/ab_env.py --op logp --rows 32768 --variants DEFAULT --rounds 1 --reps 1 > $out/${tag}_ncu_f1.log 2>&1
  echo "ncu_f1=$?" >> $st
  # f2: the fused LM-head log-prob (d = 5120, the 32B model's hidden size) and the backward GEMMs (8192-row chunk)
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:lmhead_tile -s 1 -c 1 -o $out/${tag}_f2 \
      python tools/ab_env.py --op lm --rows 32768 --d 5120 --variants DEFAULT --rounds 1 --reps 1 > $out/${tag}_ncu_f2.log 2>&1
  echo "ncu_f2=$?" >> $st
  for op in dh dw; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tile -s 1 -c 1 -o $out/${tag}_gemm_$op \
        python tools/ab_env.py --op $op --rows 8192 --d 5120 --variants DEFAULT --rounds 1 --reps 1 > $out/${tag}_ncu_gemm_$op.log 2>&1
    echo "ncu_gemm_$op=$?" >> $st
  done
fi
cat $st
