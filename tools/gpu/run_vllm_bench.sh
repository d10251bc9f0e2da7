#!/bin/bash
# vLLM+ (NEXT-2) bench line + launch list + one full ncu capture of replay_kernel<1>
mkdir -p gpurun_out
timeout 1200 python bench.py --policy vllm --steps 5 --warmup 3 > gpurun_out/bench_vllm.jsonl 2> gpurun_out/bench_vllm.err; echo "bench rc=$?"
tail -1 gpurun_out/bench_vllm.jsonl | cut -c1-1500
tail -3 gpurun_out/bench_vllm.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_vllm.csv \
  python bench.py --policy vllm --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_vllm_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o gpurun_out/prof_replay_vllm python bench.py --policy vllm --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_vllm.log 2>&1; echo "full rc=$?"
