#!/bin/bash
mkdir -p gpurun_out
for nw in 2368 148; do for f in build/variants/*.so; do
  NW=$nw PHASES4=1 MARCONI_LIB=$PWD/$f timeout 600 python tools/variant_timing.py 2>&1 | tail -2
done; done | tee gpurun_out/nw.txt
