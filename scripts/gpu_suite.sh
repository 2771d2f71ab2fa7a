# build, smoke, full GPU parity suite, bench lines for all configs
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -15 gpurun_out/pytest_gpu.log
for spec in "c3 dac auto" "c3 ccf auto" "c3 binary auto" "c2 dac auto" "c1 dac auto" "c4 dac auto" "c5 dac auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline \
    > gpurun_out/bench_$1_$2_$3.json 2> gpurun_out/bench_$1_$2_$3.err; echo bench $spec rc=$?
  python scripts/summarize.py gpurun_out/bench_$1_$2_$3.json
done
if [ -n "$LAUNCHES" ]; then
for cfg in $LAUNCHES; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$cfg.csv python bench.py --config $cfg --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$cfg.log 2>&1; echo launches $cfg rc=$?
python scripts/ncu_summary.py --launches gpurun_out/launches_$cfg.json gpurun_out/launches_$cfg.csv
python -c "
import json; d=json.load(open('gpurun_out/launches_$cfg.json'))
for k,v in d['per_kernel'].items(): print('$cfg', k[:60], v['launches'], round(v['us']/v['launches'],1))"
done
fi
