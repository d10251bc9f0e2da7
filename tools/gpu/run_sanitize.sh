#!/bin/bash
# compute-sanitizer passes over the smoke replay and one micro-trace parity test
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.log 2>&1; echo "$tool smoke rc=$?"
  tail -3 gpurun_out/san_$tool.log
done
timeout 1200 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "scenarios_on_gpu or eviction_examples or chunked_paper or vllm_occurrence" > gpurun_out/san_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"
tail -3 gpurun_out/san_memcheck_tests.log
