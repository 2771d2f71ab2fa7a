# build, dac/fused parity tests, three c3 dac bench lines (the headline)
mkdir -p gpurun_out/c3
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "dac or fused or graph" > gpurun_out/c3/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/c3/pytest.log
for i in 1 2 3; do
timeout 300 python bench.py --config c3 --sampler dac --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c3/bench_c3_$i.json 2> gpurun_out/c3/bench_c3_$i.err; echo bench rc=$?
python scripts/summarize.py gpurun_out/c3/bench_c3_$i.json
done
