# build, GPU parity suite, table-build timings (bench table_build key) for c2 / c3 / c5
mkdir -p gpurun_out/k1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/k1/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/k1/pytest.log
for cfg in c3 c5 c2; do
  timeout 300 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/k1/bench_$cfg.json 2> gpurun_out/k1/bench_$cfg.err; echo bench $cfg rc=$?
  python -c "
import json; d=json.loads(open('gpurun_out/k1/bench_$cfg.json').read().strip().splitlines()[-1]); tb=d.get('table_build') or {}
print('$cfg', 'step', round(d['ms_per_step']*1e3,2), 'us; table_build', round(tb.get('ms',0)*1e3,1), 'us', round(tb.get('GB/s',0)), 'GB/s frac', round(tb.get('frac',0),3))"
done
