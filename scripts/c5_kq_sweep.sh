# c5 index-search sweep over MATCH_KQ (u's per thread); rebuilds libdrs.so per value, restores the default at the end
for kq in 2 8; do
  make -C paper_2604_01356_b200/csrc -s clean > /dev/null 2>&1
  make -C paper_2604_01356_b200/csrc -s NVFLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -DMATCH_KQ=$kq" > /dev/null 2>&1
  timeout 600 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/b.json 2>/dev/null
  echo kq=$kq; python scripts/summarize.py /tmp/b.json
done
# restore the default build
make -C paper_2604_01356_b200/csrc -s clean > /dev/null 2>&1
make -C paper_2604_01356_b200/csrc -s > /dev/null 2>&1
