#!/bin/bash
run() { f=$1; shift; echo "== $f $*"; env "$@" MARCONI_LIB=$PWD/build/variants/$f CFG=${CFG:-3} timeout 300 python tools/variant_timing.py 2>&1 | tail -1; }
for i in 1 2; do
run base.so A=1
run base.so SMEMN=32
run base.so SMEMN=512
run base.so SMEMN=1024
done
