#!/bin/bash
# round evidence: GPU parity suite, smoke, bench lines (config 3 default; 4; 4 copy layout; 5),
# launch list of the default bench, one full ncu capture of replay_kernel for config 3 and config 4 copy
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --timeout=900 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.jsonl | cut -c1-200
for a in "4" "4 --layout copy" "5"; do
  n=$(echo $a | tr -d ' -'); timeout 1200 python bench.py --config $a --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$n.jsonl 2> gpurun_out/bench_cfg$n.err; echo "cfg $a rc=$?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --no-traffic > gpurun_out/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o gpurun_out/prof_replay python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-traffic > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o gpurun_out/prof_replay_cfg4copy python bench.py --config 4 --layout copy --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --no-traffic > gpurun_out/ncu_full4.log 2>&1; echo "full4 rc=$?"
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2.jsonl 2> gpurun_out/bench_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --policy vllm --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_vllm.jsonl 2> gpurun_out/bench_vllm.err; echo "vllm rc=$?"
