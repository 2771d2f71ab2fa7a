#!/bin/bash
# Round-2 measurement set: bench lines for every config, the ncu launch list of
# the default bench, full captures of the dominant kernels; summaries in $OUT
# (gpurun_out/, copied to profiles/r2 afterwards).
cd $GRAFT_REPO_ROOT
OUT=${OUT:-gpurun_out/r2p}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1; echo build rc=$?
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo bench rc=$?
python scripts/summarize.py $OUT/bench_default.json
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_ref.err; echo ref rc=$?
for spec in "c3 ccf auto" "c3 dac merge" "c3 binary auto" "c2 dac auto" "c2 ccf auto" "c1 dac auto" "c4 dac auto" "c5 dac auto" "c5 ccf auto" "c5 binary auto"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-scaling-blocks \
    > $OUT/bench_$1_$2_$3.json 2> $OUT/bench_$1_$2_$3.err; echo bench $spec rc=$?
  python scripts/summarize.py $OUT/bench_$1_$2_$3.json
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches_c3.csv $CMD > $OUT/ncu_launch.log 2>&1; echo launches rc=$?
python scripts/ncu_summary.py --launches $OUT/launches_c3_dac.json $OUT/launches_c3.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dac_fused" -s 3 -c 1 -o $OUT/full_c3_fused $CMD > $OUT/ncu1.log 2>&1; echo full1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 1 -o $OUT/full_c3_merge python bench.py --sampler ccf --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks > $OUT/ncu2.log 2>&1; echo full2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resample_batched|k_batched_uniforms" -s 4 -c 2 -o $OUT/full_c4_batched python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-parity > $OUT/ncu3.log 2>&1; echo full3 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_unif_pass|k_chain|k_merge_tiles|k_unif_fin" -s 6 -c 5 -o $OUT/full_c2 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-graph > $OUT/ncu4.log 2>&1; echo full4 rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_match_index_sm" -s 2 -c 1 -o $OUT/full_c5_search python bench.py --config c5 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-graph > $OUT/ncu5.log 2>&1; echo full5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table_pass|k_chain_groups" -s 3 -c 3 -o $OUT/full_c3_table python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks --no-graph > $OUT/ncu6.log 2>&1; echo full6 rc=$?
python scripts/ncu_summary.py $OUT/ncu_full.json $OUT/full_c3_fused.ncu-rep $OUT/full_c3_merge.ncu-rep $OUT/full_c4_batched.ncu-rep $OUT/full_c2.ncu-rep $OUT/full_c5_search.ncu-rep $OUT/full_c3_table.ncu-rep
for r in full_c3_fused full_c3_merge full_c4_batched full_c2 full_c5_search full_c3_table; do python scripts/ncu_src.py $OUT/$r.ncu-rep "" 25 > $OUT/lines_$r.txt 2>&1; done
timeout 600 python scripts/shard_rank_time.py > $OUT/shard_rank_time_c5.json 2> $OUT/shard.err; echo shard rc=$?
timeout 600 python scripts/bench_extras.py > $OUT/bench_extras.json 2> $OUT/extras.err; echo extras rc=$?
rm -f $OUT/*.ncu-rep.bak
ls -la $OUT | head -60
