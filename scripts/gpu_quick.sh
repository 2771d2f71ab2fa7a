# quick GPU check: build, parity tests, a few bench lines
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
for spec in ${BENCH_SPECS:-"c3 dac auto" "c4 dac auto"}; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline \
    > gpurun_out/bench_$1_$2_$3.json 2> gpurun_out/bench_$1_$2_$3.err; echo bench $spec rc=$?
  python scripts/summarize.py gpurun_out/bench_$1_$2_$3.json
done
