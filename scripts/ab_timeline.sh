#!/bin/bash
# per-kernel CTA timelines of one step, baseline tree (.bl) and working tree
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abtl}; mkdir -p $D
ARGS=${ARGS:-"c2 dac auto"}
(cd .bl && timeout 600 python scripts/timeline.py $ARGS > ../$D/tl_bl.txt 2>&1); echo bl rc=$?; grep -v Remark $D/tl_bl.txt | tail -12
timeout 600 python scripts/timeline.py $ARGS > $D/tl_new.txt 2>&1; echo new rc=$?; grep -v Remark $D/tl_new.txt | tail -12
