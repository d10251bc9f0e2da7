#!/bin/bash
# bench lines of the other throughput configs (SWEBench-shaped config 4, synthetic config 5)
mkdir -p gpurun_out
for cfg in 4 5; do
  timeout 1200 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$cfg.jsonl 2> gpurun_out/bench_cfg$cfg.err; echo "cfg$cfg rc=$?"
  tail -1 gpurun_out/bench_cfg$cfg.jsonl | cut -c1-400
  tail -2 gpurun_out/bench_cfg$cfg.err
done
