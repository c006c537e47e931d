python bench.py > gpurun_out/r01g_bench.json 2> gpurun_out/r01g_bench.err
python bench.py --config 5 --steps 3 --warmup 3 --no-alt --no-cpu-baseline --no-e2e > gpurun_out/r01g_bench_config5.json 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01g_smoke.log 2>&1; tail -1 gpurun_out/r01g_smoke.log
