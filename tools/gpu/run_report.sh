#!/bin/bash
# GPU tests for the report + live tuning, then the full report (-> gpurun_out/report.{md,json})
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_report.py tests/test_gpu_livetune.py -x -q > gpurun_out/pytest_report.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/pytest_report.log
timeout 1800 python -m paper_2411_19379_b200.report --json gpurun_out/report.json > gpurun_out/report.md 2> gpurun_out/report.err; echo "report rc=$?"; tail -5 gpurun_out/report.err
