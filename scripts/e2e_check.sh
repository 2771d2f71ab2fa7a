#!/bin/bash
# GPU suite (samplers), the host-overhead probe and the default bench line
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-e2e}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $D/smoke.log 2>&1; echo smoke rc=$?; tail -1 $D/smoke.log
timeout 1200 python -m pytest -m gpu -x -q -p no:cacheprovider ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_edge_cases.py tests/test_gpu_extras.py} > $D/pytest.log 2>&1; echo pytest rc=$?; tail -2 $D/pytest.log
timeout 300 python scripts/host_overhead_probe.py > $D/host_overhead.txt 2>&1; echo probe rc=$?; cat $D/host_overhead.txt | grep -v Remark
DRS_NO_GRAPH=1 timeout 300 python scripts/host_overhead_probe.py > $D/host_overhead_nograph.txt 2>&1; echo probe nograph rc=$?; grep "dr_sample_dac\|public\|launch +" $D/host_overhead_nograph.txt
timeout 900 python bench.py > $D/bench_default.json 2> $D/bench_default.err; echo bench rc=$?
python scripts/summarize.py $D/bench_default.json
