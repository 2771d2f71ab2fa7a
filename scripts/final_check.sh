#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2z
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2z/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2z/smoke.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2z/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/r2z/gpu_tests.log
timeout 900 python scripts/run_reference_suite.py --out gpurun_out/r2z/reference_suite.txt > /dev/null 2>&1; echo "refsuite rc=$?"; tail -2 gpurun_out/r2z/reference_suite.txt
timeout 900 python bench.py > gpurun_out/r2z/bench_default.json 2> gpurun_out/r2z/bench_default.err; echo "bench rc=$?"
python scripts/summarize.py gpurun_out/r2z/bench_default.json
timeout 900 python bench.py --impl reference > gpurun_out/r2z/bench_reference.json 2> gpurun_out/r2z/bench_reference.err; echo "ref rc=$?"; tail -c 400 gpurun_out/r2z/bench_reference.json
