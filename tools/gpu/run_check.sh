#!/bin/bash
# GPU parity suite + smoke + bench line (no profiler)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -2 gpurun_out/smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.jsonl
