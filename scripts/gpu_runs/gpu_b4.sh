python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/r01f_bench_config4.json 2> gpurun_out/r01f_bench_config4.err
tail -c 1500 gpurun_out/r01f_bench_config4.json; tail -5 gpurun_out/r01f_bench_config4.err
