#!/bin/bash
# A/B of the small-n sorted uniforms: one cooperative launch (default) against
# the four-launch pipeline (DRS_NO_FUSED_UNIFORMS=1), c3 ccf / dac merge and c1
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-uab}; mkdir -p $D
for v in fused pipe; do
  if [ $v = pipe ]; then export DRS_NO_FUSED_UNIFORMS=1; else unset DRS_NO_FUSED_UNIFORMS; fi
  for spec in "c3 ccf auto" "c3 dac merge" "c1 ccf auto" "c3 dac auto"; do
    set -- $spec
    timeout 600 python bench.py --config $1 --sampler $2 --mode $3 --steps 20 --warmup 5 --no-cpu-baseline --no-scaling-blocks --no-parity \
      > $D/${v}_$1_$2_$3.json 2> $D/${v}_$1_$2_$3.err; echo "$v $spec rc=$?"
  done
done
python scripts/summarize.py $D/*.json
