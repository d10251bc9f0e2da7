#!/bin/bash
# A/B timing of build/variants/*.so, then an ncu source-counter capture (per-SASS instruction
# execution counts, warp-stall samples) of one replay launch for the variants in $SRC
mkdir -p gpurun_out
ROUNDS=${ROUNDS:-2} ./tools/gpu/run_ab_quick.sh
for n in $SRC; do
  MARCONI_LIB=$PWD/build/variants/$n.so timeout 900 ncu --section SourceCounters --section WarpStateStats --clock-control none \
    --import-source on -k regex:replay_kernel -s 1 -c 1 -o gpurun_out/src_$n python tools/variant_timing.py > gpurun_out/ncusrc_$n.log 2>&1
  echo "$n rc=$?"
done
