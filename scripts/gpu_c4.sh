mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k batched > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
CMD="python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline"
$CMD > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo bench rc=$?; python scripts/summarize.py gpurun_out/bench_c4.json; tail -3 gpurun_out/bench_c4.err
CMD="python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resample_batched" -s 2 -c 1 -o gpurun_out/prof_c4 $CMD > gpurun_out/ncu_c4.log 2>&1; echo ncu rc=$?
