#!/bin/bash
mkdir -p gpurun_out
for f in build/variants/*.so; do
  b=$(basename $f .so)
  MARCONI_LIB=$PWD/$f CFG=3 DUMP=gpurun_out/dist_$b.npz timeout 600 python tools/variant_timing.py 2>&1 | head -1
done
