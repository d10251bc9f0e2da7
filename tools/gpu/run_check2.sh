#!/bin/bash
# new GPU tests + full GPU suite + bench line (config 3) with the traffic probe
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_e2e.py -x -q > gpurun_out/pytest_e2e.log 2>&1; echo "e2e tests rc=$?"; tail -15 gpurun_out/pytest_e2e.log
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
