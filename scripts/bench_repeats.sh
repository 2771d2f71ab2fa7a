#!/bin/bash
# run-to-run spread of the headline line: the default bench five times on one box
cd $GRAFT_REPO_ROOT
OUT=${OUT:-gpurun_out/r2v}
mkdir -p $OUT
for i in 1 2 3 4 5; do
  timeout 600 python bench.py --no-scaling-blocks --no-parity --cpu-seconds 2 > $OUT/rep_$i.json 2>/dev/null; echo "rep $i rc=$?"
done
python - <<'PY'
import json, glob, statistics, os
out = os.environ.get("OUT", "gpurun_out/r2v")
rows = []
for f in sorted(glob.glob(f"{out}/rep_*.json")):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    rows.append((d["ms_per_step"] * 1e3, d["e2e"]["ms_per_step"] * 1e3, d["roofline"]["kernel_ms"] * 1e3,
                 d["table_build"]["ms"] * 1e3, d["filter_step"]["ms"] * 1e3))
names = ["step_us", "e2e_us", "kernel_us", "table_build_us", "filter_step_us"]
res = {n: {"median": statistics.median(c), "min": min(c), "max": max(c)} for n, c in zip(names, zip(*rows))}
json.dump({"runs": len(rows), "config": "c3 dac auto (default bench), one B200", **res}, open(f"{out}/spread.json", "w"), indent=1)
print(json.dumps(res, indent=1))
PY
