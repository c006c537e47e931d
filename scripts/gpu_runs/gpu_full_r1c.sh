timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
python bench.py > gpurun_out/b_main.json 2> gpurun_out/b_main.err; cat gpurun_out/b_main.json
python bench.py --config 5 --steps 3 --warmup 3 --no-alt --no-cpu-baseline --no-e2e > gpurun_out/b_c5.json 2>&1; tail -c 600 gpurun_out/b_c5.json
