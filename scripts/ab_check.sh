#!/bin/bash
# A/B on one box: the committed baseline tree (.bl) against the working tree
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-ab}; mkdir -p $D
shift
CFGS=${CFGS:-"c2 c3"}
summ() {
python - "$1" <<'PY'
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); tb=d.get('table_build') or {}
print(sys.argv[1].split('/')[-1], 'step', round(d['ms_per_step']*1e3,2), 'us kern', round(d['roofline']['kernel_ms']*1e3,2), 'e2e', round(d['e2e'].get('ms_per_step', 0)*1e3,1), 'K1', round(tb.get('ms',0)*1e3,1), 'two-pass', round(tb.get('two_pass_ms',0)*1e3,1))
PY
}
for rep in 1 2; do
for cfg in $CFGS; do
  (cd .bl && timeout 600 python bench.py --config $cfg --steps 30 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks $EXTRA > ../$D/bl_${cfg}_$rep.json 2> ../$D/bl_${cfg}_$rep.err); summ $D/bl_${cfg}_$rep.json
  for tb in deferred two-pass; do
    timeout 600 python bench.py --config $cfg --table $tb --steps 30 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks $EXTRA > $D/new_${cfg}_${tb}_$rep.json 2> $D/new_${cfg}_${tb}_$rep.err; summ $D/new_${cfg}_${tb}_$rep.json
  done
done
done
