#!/bin/bash
# fused resample + gather: parity tests, then the bench's resample_gather block (c1, c3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2g
timeout 600 python -m pytest tests/test_gpu_gather_fused.py tests/test_gpu_extras.py -q -m gpu > gpurun_out/r2g/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/r2g/tests.log
for c in c3 c1 c2; do
  timeout 600 python bench.py --config $c --no-scaling-blocks > gpurun_out/r2g/bench_$c.json 2> gpurun_out/r2g/bench_$c.err; echo "bench $c rc=$?"
  python -c "import json,sys; d=json.loads(open('gpurun_out/r2g/bench_$c.json').read().strip().splitlines()[-1]); print('$c', d['value'], d['ms_per_step'], d.get('resample_gather'))"
done
