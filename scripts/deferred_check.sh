#!/bin/bash
# the deferred (single-pass) table: parity tests, then K1 / headline / c5 lines
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-deferred}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $D/smoke.log
timeout 1500 python -m pytest tests/test_gpu_deferred.py tests/test_gpu_parity.py tests/test_gpu_extras.py tests/test_gpu_edge_cases.py -q -x -p no:cacheprovider > $D/tests.log 2>&1; echo "tests rc=$?"; tail -15 $D/tests.log
for cfg in c3 c2; do
  timeout 600 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-parity > $D/bench_$cfg.json 2> $D/bench_$cfg.err; echo bench $cfg rc=$?
  python - <<PY
import json; d=json.loads(open('$D/bench_$cfg.json').read().strip().splitlines()[-1]); tb=d.get('table_build') or {}; fs=d.get('filter_step') or {}
print('$cfg', 'step', round(d['ms_per_step']*1e3,2), 'us e2e', d['e2e']['value'], '; K1', round(tb.get('ms',0)*1e3,1), 'us frac', round(tb.get('frac',0),3), 'two-pass', round(tb.get('two_pass_ms',0)*1e3,1), 'us; filter step', round(fs.get('ms',0)*1e3,1), 'us')
PY
done
