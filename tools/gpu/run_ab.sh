#!/bin/bash
# GPU parity suite (unless NOTEST=1), then A/B timing of build/variants/*.so on config CFG (default 3)
mkdir -p gpurun_out
if [ -z "$NOTEST" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
  tail -3 gpurun_out/pytest_gpu.log
fi
for i in 1 2; do
for f in build/variants/*.so; do
  MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -1
done; done | tee gpurun_out/variants.txt
