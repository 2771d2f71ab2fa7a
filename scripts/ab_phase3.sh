#!/bin/bash
cd $GRAFT_REPO_ROOT
D=gpurun_out/${1:-abph}; mkdir -p $D
for r in 1 2; do
  (cd .bl && timeout 300 python scripts/phase_times.py c3 > ../$D/p_bl_$r.txt 2>&1); echo "== bl"; grep -v Remark $D/p_bl_$r.txt | tail -12
  DRS_TABLE=two-pass DRS_PROF_FLAGS="-DDRS_EXP_NOPPREF" timeout 300 python scripts/phase_times.py c3 > $D/p_tp_$r.txt 2>&1; echo "== tp"; grep -v Remark $D/p_tp_$r.txt | tail -12
done
