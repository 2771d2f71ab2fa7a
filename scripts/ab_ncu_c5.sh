#!/bin/bash
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abncu}; mkdir -p $D
CMD="python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks --no-graph"
(cd .bl && timeout 900 ncu --set full --clock-control none -k regex:"k_match_index_sm" -s 2 -c 1 -o ../$D/bl $CMD > ../$D/bl.log 2>&1); echo bl rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_match_index_sm" -s 2 -c 1 -o $D/new $CMD > $D/new.log 2>&1; echo new rc=$?
python scripts/ncu_summary.py $D/sum.json $D/bl.ncu-rep $D/new.ncu-rep
python - <<PY
import json; d=json.load(open("$D/sum.json"))
for k,v in d.items():
    for r in v: print(k, r["kernel"][:50], round(r["duration_us"],1), "regs", r.get("launch__registers_per_thread"), "grid", r.get("launch__grid_size"), "inst", r.get("smsp__inst_executed.sum"), "dram", round(r["dram_bytes"]/1e9,3), "warps", r.get("sm__warps_active.avg.pct_of_peak_sustained_active"))
PY
