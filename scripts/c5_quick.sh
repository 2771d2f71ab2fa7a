# build, GPU parity suite, c5 bench line (MATCH_KQ sweep with KQ=... set at build)
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_c5.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_c5.log
timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo bench rc=$?
python scripts/summarize.py gpurun_out/bench_c5.json
