# bench lines for every config + ncu launch list of the default bench + full
# captures of the dominant kernels; summaries written to $OUT (under gpurun_out/, copied to profiles/ afterwards)
OUT=${OUT:-gpurun_out/prof}
mkdir -p gpurun_out $OUT
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python bench.py > $OUT/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
python scripts/summarize.py $OUT/bench_default.json
timeout 600 python bench.py --impl reference > $OUT/bench_reference.json 2> gpurun_out/bench_ref.err; echo ref rc=$?
for spec in "c3 ccf auto" "c3 dac merge" "c3 binary auto" "c2 dac auto" "c2 ccf auto" "c1 dac auto" "c4 dac auto" "c5 dac auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline \
    > $OUT/bench_$1_$2_$3.json 2> gpurun_out/bench_$1_$2_$3.err; echo bench $spec rc=$?
  python scripts/summarize.py $OUT/bench_$1_$2_$3.json
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
python scripts/ncu_summary.py --launches $OUT/launches_c3_dac.json gpurun_out/launches_c3.csv
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dac_fused" -s 3 -c 1 -o gpurun_out/full_c3_fused $CMD > gpurun_out/ncu1.log 2>&1; echo full1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 1 -o gpurun_out/full_c3_merge python bench.py --sampler ccf --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1; echo full2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resample_batched|k_batched_uniforms" -s 4 -c 2 -o gpurun_out/full_c4_batched python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu3.log 2>&1; echo full3 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_table_pass|k_unif_pass|k_chain" -s 0 -c 8 -o gpurun_out/full_c2_scans python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu4.log 2>&1; echo full4 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 1 -o gpurun_out/full_c2_merge python bench.py --config c2 --sampler ccf --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu5.log 2>&1; echo full5 rc=$?
python scripts/ncu_summary.py $OUT/ncu_full.json gpurun_out/full_c3_fused.ncu-rep gpurun_out/full_c3_merge.ncu-rep gpurun_out/full_c4_batched.ncu-rep gpurun_out/full_c2_scans.ncu-rep gpurun_out/full_c2_merge.ncu-rep
for r in full_c3_fused full_c3_merge full_c4_batched full_c2_merge; do python scripts/ncu_src.py gpurun_out/$r.ncu-rep "" 25 > $OUT/lines_$r.txt 2>&1; done
timeout 600 python scripts/bench_extras.py > $OUT/bench_extras.json 2> gpurun_out/extras.err; echo extras rc=$?
timeout 600 python scripts/shard_rank_time.py > $OUT/shard_rank_time_c5.json 2> gpurun_out/shard.err; echo shard rc=$?
