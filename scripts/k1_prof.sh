mkdir -p gpurun_out/k1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain_groups" -s 0 -c 6 -o gpurun_out/k1/full_k1 python bench.py --config c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/k1/ncu.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/k1/ncu_full.json gpurun_out/k1/full_k1.ncu-rep
