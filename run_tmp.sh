#!/bin/bash
NOTEST=1 ./run_variants.sh
LOADT=1 MARCONI_LIB=$PWD/build/variants/lib_imglt.so python tools/variant_timing.py 2>&1 | tail -1
