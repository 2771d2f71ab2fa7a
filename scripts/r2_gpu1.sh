#!/bin/bash
# round-2 GPU check: new parity tests, box facts, bench c3 with the parity block
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2a
free -g > gpurun_out/r2a/free.txt; nproc >> gpurun_out/r2a/free.txt; nvidia-smi -L >> gpurun_out/r2a/free.txt
timeout 900 python -m pytest tests/test_gpu_c5.py -x -q -s > gpurun_out/r2a/c5.log 2>&1; echo "c5 rc=$?" >> gpurun_out/r2a/c5.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench_c3.json 2> gpurun_out/r2a/bench_c3.err
tail -3 gpurun_out/r2a/c5.log
tail -c 3000 gpurun_out/r2a/bench_c3.json
