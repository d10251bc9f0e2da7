#!/bin/bash
# round-end evidence: GPU parity suite, smoke, bench line, launch list, one full ncu capture
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout=600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.jsonl 2> gpurun_out/bench.err; echo "bench rc=$?"
tail -1 gpurun_out/bench.jsonl | cut -c1-200
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; echo "launches rc=$?"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:replay_kernel -s 1 -c 1 \
  -o gpurun_out/prof_replay python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "full rc=$?"
for cfg in 4 5; do
  timeout 1200 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$cfg.jsonl 2> gpurun_out/bench_cfg$cfg.err; echo "cfg$cfg rc=$?"
done
