for occ in 4 5; do
  sed -i "s/__global__ void __launch_bounds__(UW_FILTERS \* LANES, [0-9]) k_batched_uniforms_warp/__global__ void __launch_bounds__(UW_FILTERS * LANES, $occ) k_batched_uniforms_warp/" paper_2604_01356_b200/csrc/drs_batched.cu
  make -C paper_2604_01356_b200/csrc -s > /dev/null 2>&1
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_batched_uniforms" -c 3 --csv python bench.py --config c4 --steps 2 --warmup 1 --no-cpu-baseline 2>/dev/null | grep -i "uniforms" | tail -1 | awk -F'","' '{print "occ='$occ'", $NF}'
done
