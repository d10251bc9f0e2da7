#!/bin/bash
# A/B timing of build/variants/*.so, then per variant a few ncu metrics of one replay launch
# (instructions, issue activity, stall ratios, L2 hit rate)
mkdir -p gpurun_out
ROUNDS=${ROUNDS:-2} ./tools/gpu/run_ab_quick.sh
M=smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,gpu__time_duration.sum
for f in build/variants/*.so; do case $f in *t3*) continue;; esac
  n=$(basename $f .so)
  MARCONI_LIB=$PWD/$f timeout 600 ncu --metrics $M --clock-control none -k regex:replay_kernel -s 1 -c 1 --csv \
    python tools/variant_timing.py > gpurun_out/ncum_$n.csv 2>&1; echo "$n rc=$?"
  grep -E '"(smsp|lts|l1tex|gpu)__' gpurun_out/ncum_$n.csv | awk -F'","' '{print $(NF-2), $NF}' | sed "s/^/$n /"
done
