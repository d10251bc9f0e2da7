#!/bin/bash
mkdir -p gpurun_out
for f in build/variants/*.so; do
  MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -1
done | tee gpurun_out/variants.txt
