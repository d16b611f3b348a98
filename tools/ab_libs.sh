#!/bin/bash
# A/B several builds of libecho.so on the same box: bash tools/ab_libs.sh tag lib1 lib2 ...
# (AB_CMD overrides the measured command; default: tools/prof_kernel.py over $ALGOS)
tag=$1; shift
cp paper_2508_05387_b200/libecho.so /tmp/libecho_orig.so
for lib in "$@"; do
  cp $lib paper_2508_05387_b200/libecho.so
  touch paper_2508_05387_b200/libecho.so
  echo "== $lib" >> gpurun_out/${tag}_ab.log
  timeout 300 ${AB_CMD:-python tools/prof_kernel.py --algos ${ALGOS:-quad_reg}} >> gpurun_out/${tag}_ab.log 2>&1
done
cp /tmp/libecho_orig.so paper_2508_05387_b200/libecho.so
