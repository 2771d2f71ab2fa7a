#!/bin/bash
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2i
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_unif_pass1" -s 6 -c 1 -o gpurun_out/r2i/full_pass1 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-scaling-blocks --no-graph > gpurun_out/r2i/ncu1.log 2>&1; echo full1 rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_batched_uniforms" -s 4 -c 1 -o gpurun_out/r2i/full_bunif python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-parity --no-graph > gpurun_out/r2i/ncu2.log 2>&1; echo full2 rc=$?
ls -la gpurun_out/r2i
