#!/bin/bash
# merge tiles: per-u bisection (default) against the linear merge path from 64 u's per tile (DRS_MERGE_PATHS_MIN=64)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-mab}; mkdir -p $D
for v in bisect paths64; do
  if [ $v = paths64 ]; then export DRS_MERGE_PATHS_MIN=64; else unset DRS_MERGE_PATHS_MIN; fi
  for spec in "c2 dac auto" "c2 ccf auto" "c3 ccf auto" "c5 ccf auto" "c5 dac merge" "c1 ccf auto"; do
    set -- $spec
    timeout 600 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-scaling-blocks --no-parity \
      > $D/${v}_$1_$2_$3.json 2> $D/${v}_$1_$2_$3.err; echo "$v $spec rc=$?"
  done
done
python scripts/summarize.py $D/*.json
