#!/bin/bash
# full captures of k_merge_tiles on the final tree (24 KB tiles at M >> N): c3 ccf and c5 ccf
cd $GRAFT_REPO_ROOT
OUT=${OUT:-gpurun_out/r2m}; mkdir -p $OUT
A="--steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks"
python bench.py --sampler ccf $A > /dev/null 2>&1; echo plain rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 3 -c 1 -o $OUT/full_c3_merge python bench.py --sampler ccf $A > $OUT/ncu_c3.log 2>&1; echo c3 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles|k_merge_heavy" -s 6 -c 2 -o $OUT/full_c5_merge python bench.py --config c5 --sampler ccf $A > $OUT/ncu_c5.log 2>&1; echo c5 rc=$?
python scripts/ncu_summary.py $OUT/ncu_merge_tiles_final.json $OUT/full_c3_merge.ncu-rep $OUT/full_c5_merge.ncu-rep
python scripts/ncu_src.py $OUT/full_c5_merge.ncu-rep "k_merge_tiles" 20 > $OUT/lines_full_c5_merge.txt 2>&1
rm -f $OUT/*.ncu-rep
cat $OUT/ncu_merge_tiles_final.json | head -c 3000
