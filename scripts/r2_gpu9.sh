#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2h
for spec in "c2 dac auto" "c3 ccf auto" "c5 ccf auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > gpurun_out/r2h/bench_$1_$2.json 2>/dev/null; python scripts/summarize.py gpurun_out/r2h/bench_$1_$2.json
done
