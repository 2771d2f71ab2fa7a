#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2e
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2e/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2e/gpu_tests.log
tail -3 gpurun_out/r2e/gpu_tests.log
for spec in "c2 dac auto" "c5 dac auto" "c3 ccf auto"; do
  timeout 300 python scripts/timeline.py $spec 2>&1 | grep -v "warning\|Remark\|^ *$\|\^\|constexpr" > gpurun_out/r2e/tl_${spec// /_}.txt; cat gpurun_out/r2e/tl_${spec// /_}.txt | tail -10
done
for cfg in c2 c3; do timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > gpurun_out/r2e/bench_$cfg.json 2>/dev/null; python scripts/summarize.py gpurun_out/r2e/bench_$cfg.json; done
timeout 300 python bench.py --config c3 --sampler ccf --steps 20 --warmup 5 --no-cpu-baseline --no-parity > gpurun_out/r2e/bench_c3_ccf.json 2>/dev/null; python scripts/summarize.py gpurun_out/r2e/bench_c3_ccf.json
