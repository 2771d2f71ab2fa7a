mkdir -p gpurun_out/c2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles|k_unif_pass|k_chain|k_unif_fin" -s 8 -c 5 -o gpurun_out/c2/full_c2 python bench.py --config c2 --sampler ccf --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c2/ncu.log 2>&1; echo full rc=$?
python scripts/ncu_summary.py gpurun_out/c2/ncu_full.json gpurun_out/c2/full_c2.ncu-rep
