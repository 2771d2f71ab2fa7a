mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_dac.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_c3_dac.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?
$CMD > gpurun_out/plain_dac2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_match_index|k_unif_pass|k_merge_tiles" -s 6 -c 6 -o gpurun_out/prof_c3_dac $CMD > gpurun_out/ncu_full.log 2>&1; echo full rc=$?
CMD2="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --sampler ccf"
$CMD2 > gpurun_out/plain_ccf.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_merge_tiles" -s 2 -c 2 -o gpurun_out/prof_c3_ccf $CMD2 > gpurun_out/ncu_full_ccf.log 2>&1; echo fullccf rc=$?
