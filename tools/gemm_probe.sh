#!/bin/bash
# GEMM A/B session (under gpurun): libecho's tcgen05 GEMM vs cuBLAS (fp32 out) at the f2 backward shapes, then one
# ncu --set full capture per product for both implementations.  Usage: bash tools/gemm_probe.sh <tag> [rows...]
tag=${1:-g}
shift
rows=${@:-8192 32768}
out=gpurun_out
mkdir -p $out
python -c "import __graft_entry__ as g; g.build()" > $out/${tag}_build.log 2>&1
for r in $rows; do
  for d in 2560 5120; do
    timeout 300 python tools/prof_gemm.py --rows $r --d $d --reps 5 >> $out/${tag}_prof.jsonl 2>> $out/${tag}_prof.err
  done
done
if [ "${NCU:-1}" = "1" ]; then
  for arm in dh_tc dw_tc dh_cublas dw_cublas; do
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm|nvjet|xmma|cutlass|sm100" -s 1 -c 1 -o $out/${tag}_${arm} \
      python tools/prof_gemm.py --rows 8192 --reps 1 --only $arm > $out/${tag}_ncu_${arm}.log 2>&1
    ncu -i $out/${tag}_${arm}.ncu-rep --page raw --csv > $out/${tag}_${arm}_raw.csv 2>/dev/null
  done
fi
echo done
