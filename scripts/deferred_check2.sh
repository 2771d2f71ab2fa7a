#!/bin/bash
# deferred tables: parity module, then A/B sampler lines (deferred vs two-pass table) and phase stamps
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-deferred2}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $D/smoke.log
timeout 900 python -m pytest tests/test_gpu_deferred.py -q -x -p no:cacheprovider --timeout 300 > $D/tests.log 2>&1; echo "tests rc=$?"; tail -15 $D/tests.log
summ() {
python - "$1" <<'PY'
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); tb=d.get('table_build') or {}; fs=d.get('filter_step') or {}
print(sys.argv[1].split('/')[-1], 'step', round(d['ms_per_step']*1e3,2), 'us kern', round(d['roofline']['kernel_ms']*1e3,2), 'e2e', round(d['e2e'].get('ms_per_step', 0)*1e3 if 'ms_per_step' in d['e2e'] else 0,1), '; K1', round(tb.get('ms',0)*1e3,1), 'frac', round(tb.get('frac',0),3), 'two-pass', round(tb.get('two_pass_ms',0)*1e3,1), '; filter', round(fs.get('ms',0)*1e3,1))
PY
}
for cfg in c3 c2; do
 for tb in deferred two-pass; do
  timeout 600 python bench.py --config $cfg --table $tb --steps 30 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > $D/bench_${cfg}_$tb.json 2> $D/bench_${cfg}_$tb.err; echo bench $cfg $tb rc=$?
  summ $D/bench_${cfg}_$tb.json
 done
done
for tb in deferred two-pass; do
  DRS_TABLE=$tb timeout 300 python scripts/phase_times.py c3 > $D/phase_c3_$tb.txt 2>&1; echo phase $tb rc=$?; tail -14 $D/phase_c3_$tb.txt
done
