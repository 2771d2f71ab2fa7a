#!/bin/bash
# fused-kernel phase stamps (c3), committed baseline tree (.bl) vs the working tree (two-pass and deferred tables)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abph}; mkdir -p $D
for r in 1 2 3 4; do
  (cd .bl && timeout 300 python scripts/phase_times.py c3 > ../$D/p_bl.txt 2>&1); echo "bl       $(grep 'events around' $D/p_bl.txt | sed 's/.*events around the call//')  $(grep ' 7 search' $D/p_bl.txt)  $(grep ' 8 written' $D/p_bl.txt)"
  DRS_TABLE=two-pass timeout 300 python scripts/phase_times.py c3 > $D/p_tp.txt 2>&1; echo "two-pass $(grep 'events around' $D/p_tp.txt | sed 's/.*events around the call//')  $(grep ' 7 search' $D/p_tp.txt)  $(grep ' 8 written' $D/p_tp.txt)"
  DRS_TABLE=deferred timeout 300 python scripts/phase_times.py c3 > $D/p_df.txt 2>&1; echo "deferred $(grep 'events around' $D/p_df.txt | sed 's/.*events around the call//')  $(grep ' 7 search' $D/p_df.txt)  $(grep ' 8 written' $D/p_df.txt)"
done
