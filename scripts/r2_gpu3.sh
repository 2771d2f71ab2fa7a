#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2c
timeout 1800 python -m pytest tests -m gpu -x -q -k "opstats or c4_full or stats_counted or nccl" > gpurun_out/r2c/gpu_tests_new.log 2>&1; echo "rc=$?" >> gpurun_out/r2c/gpu_tests_new.log
tail -5 gpurun_out/r2c/gpu_tests_new.log
timeout 900 python scripts/run_reference_suite.py --out gpurun_out/r2c/reference_suite.txt > /dev/null 2>&1; echo "refsuite rc=$?"
tail -15 gpurun_out/r2c/reference_suite.txt
timeout 900 python bench.py > gpurun_out/r2c/bench_default.json 2> gpurun_out/r2c/bench_default.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2c/bench_default.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['parity']['ok'], {k:(v['value'], v['ms_per_step']) for k,v in d['scaling_blocks'].items()})"
