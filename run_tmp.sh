#!/bin/bash
for m in 8192 4096 2048 8192 4096 2048; do MAXN=$m timeout 300 python tools/variant_timing.py 2>&1 | tail -1 | sed "s/^/MAXN=$m /"; done
