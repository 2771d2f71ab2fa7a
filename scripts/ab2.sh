#!/bin/bash
# A/B on one box: the committed baseline tree (.bl, a worktree of HEAD, built) against the working tree
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-ab2}; mkdir -p $D
SPECS=${SPECS:-"c4 dac auto|c2 dac auto|c3 dac auto"}
IFS='|' read -ra LIST <<< "$SPECS"
for rep in 1 2; do
for spec in "${LIST[@]}"; do
  set -- $spec
  tag=$1_$2_$3
  (cd .bl && timeout 600 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > ../$D/bl_${tag}_$rep.json 2> ../$D/bl_${tag}_$rep.err); python scripts/summarize.py $D/bl_${tag}_$rep.json
  timeout 600 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-parity --no-scaling-blocks > $D/new_${tag}_$rep.json 2> $D/new_${tag}_$rep.err; python scripts/summarize.py $D/new_${tag}_$rep.json
done
done
