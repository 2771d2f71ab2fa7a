mkdir -p gpurun_out/c2
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for smp in dac ccf; do
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file gpurun_out/c2/launches_$smp.csv python bench.py --config c2 --sampler $smp --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/c2/ncu_$smp.log 2>&1; echo $smp rc=$?
done
