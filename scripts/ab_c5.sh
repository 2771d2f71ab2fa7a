#!/bin/bash
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abc5}; mkdir -p $D
summ() {
python - "$1" <<'PY'
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1].split('/')[-1], 'step', round(d['ms_per_step']*1e3,1), 'us kern', round(d['roofline']['kernel_ms']*1e3,1))
PY
}
(cd .bl && timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks > ../$D/bl.json 2>/dev/null); summ $D/bl.json
timeout 900 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks > $D/new.json 2>/dev/null; summ $D/new.json
