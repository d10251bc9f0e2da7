#!/bin/bash
mkdir -p gpurun_out
# launch list (cold-cache, serialised) of the bench command
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
echo "launches rc=$?"
# one full capture of the dominant kernel
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o gpurun_out/prof_replay python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
# bench with cpu baseline
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_full.log 2>&1
echo "bench rc=$?"
nproc > gpurun_out/nproc.txt; lscpu | grep -i "model name" >> gpurun_out/nproc.txt
