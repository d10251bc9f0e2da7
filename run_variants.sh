#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.jsonl | cut -c1-600; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.jsonl 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref.jsonl | cut -c1-400
