#!/bin/bash
mkdir -p gpurun_out
for f in build/variants/*.so; do
  PHASES3=1 MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -2
done | tee gpurun_out/variants.txt
