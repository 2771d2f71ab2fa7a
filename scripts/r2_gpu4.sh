#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2d
timeout 1800 python -m pytest tests -m gpu -x -q -k "opstats or c4_full or stats_counted or nccl" > gpurun_out/r2d/gpu_tests_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2d/gpu_tests_new.log
tail -3 gpurun_out/r2d/gpu_tests_new.log
timeout 900 python scripts/run_reference_suite.py --out gpurun_out/r2d/reference_suite.txt > /dev/null 2>&1; echo "refsuite rc=$?"
tail -4 gpurun_out/r2d/reference_suite.txt
for spec in "c2 dac auto" "c3 dac auto" "c3 ccf auto" "c1 dac auto" "c5 dac auto"; do
  timeout 300 python scripts/timeline.py $spec > gpurun_out/r2d/tl_${spec// /_}.txt 2>&1; cat gpurun_out/r2d/tl_${spec// /_}.txt | tail -12
done
