#!/bin/bash
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
fi
for i in 1 2; do
for f in build/variants/*.so; do
  case $f in *t1*) E="PHASES=1";; *t3*) E="PHASES3=1";; *t4*) E="PHASES4=1";; *) E="";; esac
  env $E MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -2
done; done | tee gpurun_out/variants.txt
