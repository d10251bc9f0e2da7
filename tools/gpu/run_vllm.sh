#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k vllm > gpurun_out/pytest_vllm.log 2>&1; echo "vllm rc=$?" >> gpurun_out/pytest_vllm.log
tail -30 gpurun_out/pytest_vllm.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
MARCONI_LIB=$PWD/paper_2411_19379_b200/libmarconi.so timeout 300 python tools/variant_timing.py 2>&1 | tail -1
