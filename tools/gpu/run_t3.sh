#!/bin/bash
MARCONI_LIB=$PWD/build/variants/t3.so CFG=3 PHASES3A=1 CHAINS=1 timeout 600 python tools/variant_timing.py 2>&1 | tail -22
