# full GPU check: build, smoke, parity tests, bench lines, ncu launch list + full capture of the top kernel
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
cat gpurun_out/bench_default.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo benchref rc=$?
cat gpurun_out/bench_ref.json
for spec in "c3 dac merge" "c3 ccf auto" "c3 binary auto" "c2 dac auto" "c2 ccf auto" "c1 dac auto" "c4 dac auto" "c5 dac auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline \
    > gpurun_out/bench_$1_$2_$3.json 2> gpurun_out/bench_$1_$2_$3.err; echo bench $spec rc=$?
done
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3_dac.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dac_fused" -s 3 -c 2 -o gpurun_out/prof_fused_c3 $CMD > gpurun_out/ncu_fused_c3.log 2>&1; echo fullfused rc=$?
CMD2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --sampler ccf"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 2 -o gpurun_out/prof_c3_ccf $CMD2 > gpurun_out/ncu_full_ccf.log 2>&1; echo fullccf rc=$?
