#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2j
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2j/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/r2j/gpu_tests.log
tail -3 gpurun_out/r2j/gpu_tests.log
timeout 900 python bench.py > gpurun_out/r2j/bench_default.json 2> gpurun_out/r2j/bench_default.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2j/bench_default.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['parity']['ok'], d['filter_step'], d['table_build']['ms'])
print({k:(v['value'], v['ms_per_step']) for k,v in d['scaling_blocks'].items()})"
for spec in "c5 binary auto" "c5 dac auto" "c3 binary auto" "c2 dac auto" "c4 dac auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > gpurun_out/r2j/bench_$1_$2.json 2>/dev/null; python scripts/summarize.py gpurun_out/r2j/bench_$1_$2.json
done
timeout 300 python scripts/phase_times.py c3 2>&1 | grep -v "warning\|Remark\|^ *$\|\^\|constexpr\|bool site\|const int64_t Mf" | tail -18
