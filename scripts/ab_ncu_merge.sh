#!/bin/bash
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abncum}; mkdir -p $D
CMD="python bench.py --config c3 --sampler ccf --steps 2 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks --no-graph"
(cd .bl && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 1 -o ../$D/bl $CMD > ../$D/bl.log 2>&1); echo bl rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 1 -o $D/new $CMD > $D/new.log 2>&1; echo new rc=$?
python scripts/ncu_summary.py $D/sum.json $D/bl.ncu-rep $D/new.ncu-rep
python - <<PY
import json; d=json.load(open("$D/sum.json"))
for k,v in d.items():
    for r in v: print(k, round(r["duration_us"],1), "regs", r.get("launch__registers_per_thread"), "grid", r.get("launch__grid_size"), "smem", r.get("launch__shared_mem_per_block_dynamic"), "inst", r.get("smsp__inst_executed.sum"), "dram", round(r["dram_bytes"]/1e9,3), "warps", round(r.get("sm__warps_active.avg.pct_of_peak_sustained_active"),1))
PY
python scripts/ncu_src.py $D/new.ncu-rep "" 15 > $D/lines_new.txt 2>&1; python scripts/ncu_src.py $D/bl.ncu-rep "" 15 > $D/lines_bl.txt 2>&1
