#!/bin/bash
mkdir -p gpurun_out
run() { f=$1; shift; echo "== $f $*"; env "$@" MARCONI_LIB=$PWD/build/variants/$f CFG=${CFG:-3} timeout 300 python tools/variant_timing.py 2>&1 | tail -3; }
for i in 1 2; do
run w1.so A=1
run w1m14.so A=1
run w1m14r128.so A=1
run w2m7.so A=1
done
run w1t3.so PHASES3=1
