#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2g
timeout 1500 python -m pytest tests -m gpu -x -q -k "merge or ccf or exact_mode or samplers_device or heavy or c5_full or boundary_report or fused or replay or repair or zero_weight or chi" > gpurun_out/r2g/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2g/gpu_tests.log
tail -3 gpurun_out/r2g/gpu_tests.log
for spec in "c2 dac auto" "c3 ccf auto" "c5 ccf auto" "c2 ccf auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > gpurun_out/r2g/bench_$1_$2.json 2>/dev/null; python scripts/summarize.py gpurun_out/r2g/bench_$1_$2.json
done
timeout 300 python scripts/timeline.py c2 dac auto 2>&1 | grep -v "warning\|Remark\|^ *$\|\^\|constexpr\|bool site\|const int64_t Mf\|RuntimeWarn\|nanmax" | tail -8
