#!/bin/bash
# Round-2 (second session) captures: K1 single-pass vs two-pass launch list
# with DRAM bytes, full captures of the single-pass kernels; summaries in $OUT
cd $GRAFT_REPO_ROOT
OUT=${OUT:-gpurun_out/r2b}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build rc=$?
python scripts/k1_driver.py > /dev/null 2>&1; echo driver rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $OUT/launches_k1_c3.csv python scripts/k1_driver.py > $OUT/ncu_k1_launch.log 2>&1; echo launches rc=$?
python scripts/ncu_summary.py --launches $OUT/launches_k1_c3.json $OUT/launches_k1_c3.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table_local|k_table_levels|k_chain_groups|k_build_top_guide" -s 4 -c 4 \
  -o $OUT/full_k1_deferred python scripts/k1_driver.py > $OUT/ncu_k1_full.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py $OUT/ncu_full_k1.json $OUT/full_k1_deferred.ncu-rep
python scripts/ncu_src.py $OUT/full_k1_deferred.ncu-rep "k_table_local" 25 > $OUT/lines_k1_local.txt 2>&1
ls -la $OUT
