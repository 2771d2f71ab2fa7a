cd $GRAFT_REPO_ROOT
D=gpurun_out/tl1; mkdir -p $D
python -c "import __graft_entry__ as g; g.build()" > $D/build.log 2>&1
for v in new old; do
  if [ $v = old ]; then export DRS_NO_FINISH=1; else unset DRS_NO_FINISH; fi
  DRS_DEBUG=1 timeout 600 python scripts/timeline.py c2 dac search > $D/tl_c2_$v.txt 2>&1; echo $v rc=$?; grep -v Remark $D/tl_c2_$v.txt | tail -9
done
