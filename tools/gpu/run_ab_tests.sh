#!/bin/bash
# GPU parity suite on the in-tree build, then A/B of build/variants/*.so on configs 3/4 x stream/copy
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
./tools/gpu/run_ab_layouts.sh
