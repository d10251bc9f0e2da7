#!/bin/bash
# one ncu --set full capture of replay_kernel per build/variants/*.so (config CFG, default 3)
mkdir -p gpurun_out
for f in build/variants/*.so; do
  n=$(basename $f .so)
  MARCONI_LIB=$PWD/$f timeout 1200 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
    -o gpurun_out/prof_$n python tools/variant_timing.py > gpurun_out/ncu_$n.log 2>&1; echo "$n rc=$?"
done
