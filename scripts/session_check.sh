#!/bin/bash
# build, smoke, GPU suite and the default bench line; output under gpurun_out/$1
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-check}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $D/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $D/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -3 $D/gpu_tests.log
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo "bench rc=$?"
python scripts/summarize.py $D/bench_default.json
