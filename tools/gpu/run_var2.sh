#!/bin/bash
mkdir -p gpurun_out
if [ -n "$TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
fi
run() { f=$1; shift; echo "== $f $*"; env "$@" MARCONI_LIB=$PWD/build/variants/$f CFG=${CFG:-3} timeout 300 python tools/variant_timing.py 2>&1 | tail -${TAILN:-3}; }
for i in 1 2 3; do
for f in build/variants/*.so; do case $f in *t3*) continue;; esac; run $(basename $f) A=1; done
done
for f in build/variants/*t3*.so; do [ -e "$f" ] && TAILN=24 run $(basename $f) PHASES3=1 PHASES3A=1 CHAINS=1; done
