#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_e2e.py tests/test_gpu_livetune.py tests/test_multigpu.py -x -q > gpurun_out/pytest_sched.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/pytest_sched.log
timeout 1200 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.jsonl 2> gpurun_out/bench_cfg5.err; echo "cfg5 rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "cfg3 rc=$?"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.jsonl 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
timeout 1800 python bench.py --gpus 2 --config 5 --scaling strong --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5_strong2.jsonl 2> gpurun_out/bench_cfg5_strong2.err; echo "cfg5 strong x2 rc=$?"
