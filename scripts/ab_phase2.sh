#!/bin/bash
# fused-kernel phase stamps (c3): baseline tree vs working tree variants (DRS_PROF_FLAGS)
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abph}; mkdir -p $D
for r in 1 2 3; do
  (cd .bl && timeout 300 python scripts/phase_times.py c3 > ../$D/p_bl.txt 2>&1); echo "bl        $(grep 'events around' $D/p_bl.txt | sed 's/.*events around the call//')  $(grep ' 7 search' $D/p_bl.txt)"
  for fl in "" "-DDRS_EXP_NOPPREF"; do
    DRS_TABLE=two-pass DRS_PROF_FLAGS="$fl" timeout 300 python scripts/phase_times.py c3 > $D/p_tp.txt 2>&1; echo "tp [$fl] $(grep 'events around' $D/p_tp.txt | sed 's/.*events around the call//')  $(grep ' 7 search' $D/p_tp.txt)"
  done
done
