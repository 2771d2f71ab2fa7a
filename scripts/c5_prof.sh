mkdir -p gpurun_out/c5
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_match_index_sm" -s 1 -c 1 -o gpurun_out/c5/full_c5 python bench.py --config c5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c5/ncu.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/c5/ncu_full.json gpurun_out/c5/full_c5.ncu-rep
