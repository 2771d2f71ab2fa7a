#!/bin/bash
# sharded windows + repair at rank boundary + full GPU suite + multi-rank bench flow (gloo, functional only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2b
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2b/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2b/gpu_tests.log
tail -5 gpurun_out/r2b/gpu_tests.log
timeout 600 python bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --no-parity > gpurun_out/r2b/bench_g2_gloo.json 2> gpurun_out/r2b/bench_g2_gloo.err; echo "g2 rc=$?"
tail -c 1500 gpurun_out/r2b/bench_g2_gloo.json; tail -5 gpurun_out/r2b/bench_g2_gloo.err
