#!/bin/bash
# Full-size GPU-vs-oracle parity (tools/parity_full.py) for the configs given as arguments
# ("4c" = config 4 in the per-request-copy layout, "3v" = bench.py's vLLM+ sweep on config 3).
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
for c in "$@"; do
  pol=marconi; lay=stream; cfg=$c
  case $c in *c) cfg=${c%c}; lay=copy;; *v) cfg=${c%v}; pol=vllm;; esac
  timeout 3000 python tools/parity_full.py --config $cfg --layout $lay --policy $pol --out gpurun_out/parity_cfg$c.json > gpurun_out/parity_cfg$c.log 2>&1
  echo "config $c rc=$?"; tail -3 gpurun_out/parity_cfg$c.log
done
