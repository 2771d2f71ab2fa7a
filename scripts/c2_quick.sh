# build, GPU parity suite, c2 / c5 bench lines, ncu capture of the c2 merge kernel (NCU=1)
mkdir -p gpurun_out/c2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/c2/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c2/pytest.log
for spec in "c2 dac auto" "c2 ccf auto" "c5 dac auto" "c3 ccf auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c2/bench_$1_$2_$3.json 2> gpurun_out/c2/bench_$1_$2_$3.err; echo bench $spec rc=$?
  python scripts/summarize.py gpurun_out/c2/bench_$1_$2_$3.json
done
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 3 -c 1 -o gpurun_out/c2/full_c2_merge python bench.py --config c2 --sampler ccf --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c2/ncu.log 2>&1; echo full rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/c2/launches_c2.csv python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2/ncu_l.log 2>&1; echo launches rc=$?
fi
