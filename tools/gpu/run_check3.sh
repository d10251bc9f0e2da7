#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke.log
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 python -m pytest tests/test_gpu_lookup.py tests/test_gpu_e2e.py -x -q -k "micro or rejects or chain_sums or cost_feedback" > gpurun_out/san_memcheck_lookup.log 2>&1; echo "memcheck lookup/e2e rc=$?"; tail -2 gpurun_out/san_memcheck_lookup.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
