#!/bin/bash
# compute-sanitizer passes over the smoke replay and a set of small GPU tests (round 2:
# + the bulk-copy / L2-prefetch paths (long-compare alignments), the device trace check,
# the host pipeline, the bootstrap live pass)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_$tool.log 2>&1; echo "$tool smoke rc=$?"
  tail -3 gpurun_out/san_$tool.log
done
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "scenarios_on_gpu or eviction_examples or chunked_paper or vllm_occurrence or long_compare" > gpurun_out/san_memcheck_tests.log 2>&1; echo "memcheck tests rc=$?"
tail -3 gpurun_out/san_memcheck_tests.log
timeout 1800 compute-sanitizer --tool memcheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_e2e.py -x -q -k "rejects or length" > gpurun_out/san_memcheck_e2e.log 2>&1; echo "memcheck e2e rc=$?"
tail -3 gpurun_out/san_memcheck_e2e.log
timeout 1800 compute-sanitizer --tool racecheck --error-exitcode 9 --print-limit 20 \
  python -m pytest tests/test_gpu_parity.py -x -q -k "scenarios_on_gpu or long_compare" > gpurun_out/san_racecheck_tests.log 2>&1; echo "racecheck tests rc=$?"
tail -3 gpurun_out/san_racecheck_tests.log
