mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1; echo build rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_unif_pass|k_merge_tiles" -s 4 -c 3 -o gpurun_out/prof_c2 python bench.py --config c2 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_c2.log 2>&1; echo ncu c2 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_unif_pass" -s 2 -c 2 -o gpurun_out/prof_c5u python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline --no-graph > gpurun_out/ncu_c5.log 2>&1; echo ncu c5 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_dac_fused" -s 3 -c 1 -o gpurun_out/prof_c3f python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c3.log 2>&1; echo ncu c3 rc=$?
