#!/bin/bash
# A/B of k_finish_search (pass 2 + repair + search in one launch) against the
# three-launch path (DRS_NO_FINISH=1); GPU tests of the search paths first
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-finish}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1; echo build rc=$?
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_edge_cases.py} > $D/pytest.log 2>&1; echo pytest rc=$?; tail -3 $D/pytest.log
for spec in ${SPECS:-"c2 dac search" "c2 dac merge" "c5 dac auto"}; do
  set -- $spec
  for v in new old; do
    if [ $v = old ]; then export DRS_NO_FINISH=1; else unset DRS_NO_FINISH; fi
    timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-scaling-blocks > $D/bench_$1_$2_$3_$v.json 2> $D/bench_$1_$2_$3_$v.err; echo bench $spec $v rc=$?
    python scripts/summarize.py $D/bench_$1_$2_$3_$v.json
  done
done
unset DRS_NO_FINISH
