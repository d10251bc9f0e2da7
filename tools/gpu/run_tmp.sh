#!/bin/bash
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
MARCONI_LIB=$PWD/build/variants/lib_default.so CHAINS=1 python tools/variant_timing.py 2>&1 | tail -4 | head -2
MARCONI_LIB=$PWD/build/variants/lib_default.so python tools/variant_timing.py 2>&1 | tail -1
PHASES3A=1 MARCONI_LIB=$PWD/build/variants/lib_t3.so python tools/variant_timing.py 2>&1 | tail -16 | head -3
