timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
python bench.py > gpurun_out/r01d_bench.json 2> gpurun_out/r01d_bench.err; cut -c1-700 gpurun_out/r01d_bench.json
python bench.py --config 5 --steps 3 --warmup 3 --no-alt --no-cpu-baseline --no-e2e > gpurun_out/r01d_bench_c5.json 2>&1; tail -c 700 gpurun_out/r01d_bench_c5.json
S="python scripts/sweep.py"
$S --config 1 --variant implicit --T 200
LSK_TRACE=/tmp/tr.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin
