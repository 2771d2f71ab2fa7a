#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2k
timeout 1500 python -m pytest tests -m gpu -x -q -k "batched or c4_full" > gpurun_out/r2k/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2k/gpu_tests.log
tail -3 gpurun_out/r2k/gpu_tests.log
timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/r2k/bench_c4.json 2>/dev/null; python scripts/summarize.py gpurun_out/r2k/bench_c4.json
