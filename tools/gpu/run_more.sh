#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.jsonl 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
tail -1 gpurun_out/bench_cfg2.jsonl | cut -c1-300
timeout 1200 python bench.py --policy vllm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_vllm.jsonl 2> gpurun_out/bench_vllm.err; echo "vllm rc=$?"
tail -1 gpurun_out/bench_vllm.jsonl | cut -c1-300
