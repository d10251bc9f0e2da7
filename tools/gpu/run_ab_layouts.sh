#!/bin/bash
# A/B timing of build/variants/*.so on configs 3/4 x stream/copy
mkdir -p gpurun_out
for cfg in 3 4; do for lay in stream copy; do for f in build/variants/*.so; do
  CFG=$cfg LAYOUT=$lay MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -1
done; done; done | tee gpurun_out/variants.txt
