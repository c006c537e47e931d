python bench.py > gpurun_out/r01d_bench.json 2> gpurun_out/r01d_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01d_launches_config2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alt > /dev/null 2>&1
python bench.py --config 5 --steps 3 --warmup 3 --no-alt --no-cpu-baseline --no-e2e > gpurun_out/r01d_bench_config5.json 2>&1
python bench.py --impl reference > gpurun_out/r01d_bench_reference.json 2>&1
