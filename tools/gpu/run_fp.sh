#!/bin/bash
run() { f=$1; shift; echo "== $f $*"; env "$@" MARCONI_LIB=$PWD/build/variants/$f CFG=${CFG:-3} timeout 300 python tools/variant_timing.py 2>&1 | tail -1; }
for i in 1 2; do
run base.so MAXN=8192
run base.so MAXN=4096
run hs0.so MAXN=4096
run hs0.so MAXN=8192
run base.so MAXN=2048
done
