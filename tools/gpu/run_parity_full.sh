#!/bin/bash
# Full-size GPU-vs-oracle parity (tools/parity_full.py) for the configs given as arguments.
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
for c in "$@"; do
  timeout 3000 python tools/parity_full.py --config $c --out gpurun_out/parity_cfg$c.json > gpurun_out/parity_cfg$c.log 2>&1
  echo "config $c rc=$?"; tail -5 gpurun_out/parity_cfg$c.log
done
