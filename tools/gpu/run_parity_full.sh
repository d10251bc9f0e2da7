#!/bin/bash
# Full-size GPU-vs-oracle parity (tools/parity_full.py) for the configs given as arguments
# ("4c" = config 4 in the per-request-copy layout).
mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
for c in "$@"; do
  case $c in *c) cfg=${c%c}; lay=copy;; *) cfg=$c; lay=stream;; esac
  timeout 3000 python tools/parity_full.py --config $cfg --layout $lay --out gpurun_out/parity_cfg$c.json > gpurun_out/parity_cfg$c.log 2>&1
  echo "config $c rc=$?"; tail -3 gpurun_out/parity_cfg$c.log
done
