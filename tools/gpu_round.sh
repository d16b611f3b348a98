#!/bin/bash
# One GPU-box session: smoke, the GPU parity suite, the default bench, the ncu launch list and one full ncu capture.
# Usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-rX}
out=gpurun_out
mkdir -p $out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv > $out/${tag}_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $out/${tag}_smoke.log 2>&1; echo "smoke=$?" > $out/${tag}_status.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 300 --timeout_method thread -rf > $out/${tag}_pytest.log 2>&1; echo "pytest=$?" >> $out/${tag}_status.txt
timeout 600 python bench.py > $out/${tag}_bench.json 2> $out/${tag}_bench.err; echo "bench=$?" >> $out/${tag}_status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $out/${tag}_bench_ref.json 2> $out/${tag}_bench_ref.err; echo "bench_ref=$?" >> $out/${tag}_status.txt
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/${tag}_launches.csv \
      python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $out/${tag}_ncu_launch.log 2>&1; echo "ncu_launches=$?" >> $out/${tag}_status.txt
  timeout 300 python tools/prof_kernel.py --algos ${ALGO:-oct_reg} --reps 1 --warmup 1 > $out/${tag}_prof_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:policy_loss_quad -s 1 -c 1 -o $out/${tag}_kernel \
      python tools/prof_kernel.py --algos ${ALGO:-oct_reg} --reps 1 --warmup 1 > $out/${tag}_ncu_full.log 2>&1; echo "ncu_full=$?" >> $out/${tag}_status.txt
fi
cat $out/${tag}_status.txt
if [ "${NCU_F2:-1}" = "1" ]; then
  timeout 300 python tools/prof_lmhead.py --reps 1 --no-unfused > $out/${tag}_f2_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmhead_tile -s 1 -c 1 -o $out/${tag}_f2 \
      python tools/prof_lmhead.py --reps 1 --no-unfused > $out/${tag}_ncu_f2.log 2>&1; echo "ncu_f2=$?" >> $out/${tag}_status.txt
fi
if [ "${NCU_F2T:-1}" = "1" ]; then
  timeout 300 python tools/prof_lmhead.py --mode logits --rows 8192 --reps 1 > $out/${tag}_f2t_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:lmhead_tile -s 2 -c 1 -o $out/${tag}_f2_logits \
      python tools/prof_lmhead.py --mode logits --rows 8192 --reps 1 > $out/${tag}_ncu_f2t.log 2>&1; echo "ncu_f2_logits=$?" >> $out/${tag}_status.txt
fi
cat $out/${tag}_status.txt
