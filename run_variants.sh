#!/bin/bash
mkdir -p gpurun_out
for f in build/variants/*.so; do
  MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -1
done | tee gpurun_out/variants.txt
MAXN=4096 MARCONI_LIB=$PWD/build/variants/lib_u2.so timeout 300 python tools/variant_timing.py 2>&1 | tail -1 | sed 's/^/maxn4096 /'
MAXN=2048 MARCONI_LIB=$PWD/build/variants/lib_u2.so timeout 300 python tools/variant_timing.py 2>&1 | tail -1 | sed 's/^/maxn2048 /'
