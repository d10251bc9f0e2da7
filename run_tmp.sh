#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "vllm or beyond_half" 2>&1 | tail -3
NOTEST=1 ./run_variants.sh
timeout 900 python bench.py --policy vllm --steps 5 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | cut -c1-400
