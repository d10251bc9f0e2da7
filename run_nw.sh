#!/bin/bash
mkdir -p gpurun_out
for nw in 2368 592 148; do
  NW=$nw PHASES3=1 MARCONI_LIB=$PWD/build/variants/lib_t3.so timeout 600 python tools/variant_timing.py 2>&1 | tail -2
  NW=$nw PHASES=1 MARCONI_LIB=$PWD/build/variants/lib_t1.so timeout 600 python tools/variant_timing.py 2>&1 | tail -2
done | tee gpurun_out/nw.txt
