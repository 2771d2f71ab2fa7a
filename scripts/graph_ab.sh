#!/bin/bash
# default bench line with and without the graph launch of the fused kernel, interleaved on one box
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-gab}; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for r in 1 2; do
  for v in graph nograph; do
    if [ $v = nograph ]; then export DRS_NO_GRAPH=1; else unset DRS_NO_GRAPH; fi
    timeout 300 python bench.py --no-cpu-baseline --no-scaling-blocks --no-parity > $D/b_${v}_$r.json 2> $D/b_${v}_$r.err
    python scripts/summarize.py $D/b_${v}_$r.json
  done
done
