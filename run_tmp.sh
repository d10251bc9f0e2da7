#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "vllm or config3_reduced_full" 2>&1 | tail -2
NOTEST=1 ./run_variants.sh
