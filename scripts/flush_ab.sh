#!/bin/bash
# the L2 flush discipline: a write-only flush leaves ~126 MB of dirty lines for the timed kernel to write back
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-fab}; mkdir -p $D
for fl in write write+read; do
  for spec in "c3 dac auto" "c3 ccf auto" "c4 dac auto" "c2 dac auto" "c5 dac auto" "c5 ccf auto"; do
    set -- $spec
    timeout 600 python bench.py --flush $fl --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-scaling-blocks --no-parity \
      > $D/${fl}_$1_$2_$3.json 2> $D/${fl}_$1_$2_$3.err; echo "$fl $spec rc=$?"
  done
done
python scripts/summarize.py $D/*.json
python - <<'PY'
import json, glob, os
for f in sorted(glob.glob(os.path.join("gpurun_out", os.environ.get("FAB", "fab"), "*c3_dac_auto.json"))):
    d = json.load(open(f)); print(f, "K1", d["table_build"]["ms"], "filter", d["filter_step"]["ms"])
PY
