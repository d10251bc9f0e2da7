#!/bin/bash
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o gpurun_out/prof_replay2 python tools/variant_timing.py > gpurun_out/ncu_full2.log 2>&1
echo "full rc=$?"
