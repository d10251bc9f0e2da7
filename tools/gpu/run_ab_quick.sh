#!/bin/bash
# A/B timing of build/variants/*.so (bounded per run), *t3* builds with phase counters, then
# (TESTS=1) the GPU suite -- timing first, so a hanging variant costs minutes, not the call
mkdir -p gpurun_out
run() { f=$1; shift; echo "== $f $*"; env "$@" MARCONI_LIB=$PWD/build/variants/$f CFG=${CFG:-3} timeout ${TO:-120} python tools/variant_timing.py 2>&1 | tail -${TAILN:-3}; }
for i in $(seq ${ROUNDS:-3}); do
for f in build/variants/*.so; do case $f in *t3*) continue;; esac; run $(basename $f) A=1; done
done
for f in build/variants/*t3*.so; do [ -e "$f" ] && TAILN=24 run $(basename $f) PHASES3=1 PHASES3A=1; done
if [ -n "$TESTS" ]; then
timeout 1200 python -m pytest tests -m gpu -x -q --timeout=300 --timeout-method=thread -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
fi
