# build, GPU parity suite, c3 binary (latency-bound search) and c5 (throughput-bound search) bench lines
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_s.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_s.log
for spec in "c3 binary auto" "c3 dac search" "c5 dac auto"; do
  set -- $spec
  timeout 600 python bench.py --config $1 --sampler $2 --mode $3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_$1_$2_$3.json 2>/dev/null; echo bench $spec rc=$?
  python scripts/summarize.py gpurun_out/b_$1_$2_$3.json
done
