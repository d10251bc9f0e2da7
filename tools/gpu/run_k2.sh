#!/bin/bash
# long-compare parity tests, full GPU suite, A/B timing (configs 3/4 x stream/copy), config-4 copy bench line
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "long_compare or copy_layout" > gpurun_out/pytest_k2.log 2>&1; echo "k2 tests rc=$?"; tail -4 gpurun_out/pytest_k2.log
timeout 1800 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
for cfg in 3 4; do for lay in stream copy; do for f in build/variants/*.so; do
  CFG=$cfg LAYOUT=$lay MARCONI_LIB=$PWD/$f timeout 300 python tools/variant_timing.py 2>&1 | tail -1
done; done; done | tee gpurun_out/variants.txt
timeout 900 python bench.py --config 4 --layout copy --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_copy.jsonl 2> gpurun_out/bench_cfg4_copy.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_cfg4_copy.err
