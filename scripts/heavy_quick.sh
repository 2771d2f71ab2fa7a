# build, the heavy-run parity tests + full GPU suite, CCF / DaC-merge bench lines incl. c5 ccf
mkdir -p gpurun_out/hv
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "heavy" > gpurun_out/hv/pytest_heavy.log 2>&1; echo pytest heavy rc=$?; tail -3 gpurun_out/hv/pytest_heavy.log
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/hv/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/hv/pytest.log
for spec in "c3 ccf auto" "c2 dac auto" "c2 ccf auto" "c5 ccf auto" "c3 dac auto"; do
  set -- $spec
  timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/hv/b_$1_$2.json 2> gpurun_out/hv/b_$1_$2.err
  python scripts/summarize.py gpurun_out/hv/b_$1_$2.json
done
