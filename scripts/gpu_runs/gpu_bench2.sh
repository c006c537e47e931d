timeout 1500 python -m pytest tests/ -q -m gpu 2>&1 | tail -3
python bench.py > gpurun_out/bench_r1b.json 2> gpurun_out/bench_r1b.err
python bench.py --variant implicit --no-cpu-baseline > gpurun_out/bench_r1b_impl.json 2>&1
S="python scripts/sweep.py"
$S --config 3 --variant stream --n 200000 --T 20 > gpurun_out/sweep_c3.json
$S --config 4 --T 50 --cps 1 > gpurun_out/sweep_c4.json
$S --config 5 --variant implicit --n 8388608 --T 2 --reps 2 > gpurun_out/sweep_c5.json
$S --config 1 --variant stream --T 200 > gpurun_out/sweep_c1.json
cat gpurun_out/bench_r1b.json gpurun_out/bench_r1b_impl.json gpurun_out/sweep_c*.json
