#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2s
timeout 600 python scripts/sanitize_workload.py > gpurun_out/r2s/plain.log 2>&1; echo "plain rc=$?"; tail -2 gpurun_out/r2s/plain.log
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/r2s/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/r2s/$tool.log
done
