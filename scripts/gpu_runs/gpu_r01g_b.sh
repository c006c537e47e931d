python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r01g_bench_config3.json 2> gpurun_out/r01g_bench_config3.err
python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/r01g_bench_config1.json 2> gpurun_out/r01g_bench_config1.err
tail -c 300 gpurun_out/r01g_bench_config3.err
