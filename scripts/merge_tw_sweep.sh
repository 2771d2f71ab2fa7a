# CCF / merge-mode timings against the merge kernel's W tile size (DRS_MT_TW)
mkdir -p gpurun_out/mt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/mt/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/mt/pytest.log
for tw in ${TWS:-4096 8192 16384}; do  # needs a DRS_MT_TW getenv in launch_merge (removed after the sweep)
for spec in "c3 ccf auto" "c2 ccf auto" "c2 dac auto" "c5 ccf auto"; do
  set -- $spec
  DRS_MT_TW=$tw timeout 300 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/mt/b_$1_$2_$tw.json 2> gpurun_out/mt/b_$1_$2_$tw.err
  echo -n "tw $tw "; python scripts/summarize.py gpurun_out/mt/b_$1_$2_$tw.json
done; done
