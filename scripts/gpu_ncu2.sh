mkdir -p gpurun_out
for cfg in c1 c3; do
CMD="python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/plain_$cfg.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_dac_fused" -s 3 -c 2 -o gpurun_out/prof_fused_$cfg $CMD > gpurun_out/ncu_fused_$cfg.log 2>&1; echo $cfg rc=$?
done
