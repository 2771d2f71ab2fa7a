# build, batched parity tests, c4 bench (+ ncu capture of both batched kernels with NCU=1)
mkdir -p gpurun_out/c4
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "batched" > gpurun_out/c4/pytest_batched.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/c4/pytest_batched.log
timeout 300 python bench.py --config c4 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/c4/bench_c4.json 2> gpurun_out/c4/bench_c4.err; echo bench rc=$?
python scripts/summarize.py gpurun_out/c4/bench_c4.json; tail -3 gpurun_out/c4/bench_c4.err
if [ -n "$NCU" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_resample_batched|k_batched_uniforms" -s 4 -c 2 -o gpurun_out/c4/full_c4 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4/ncu.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/c4/ncu_full.json gpurun_out/c4/full_c4.ncu-rep
fi
