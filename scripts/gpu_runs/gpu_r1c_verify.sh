# re-entry verification of HEAD on a fresh box
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -5
python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err
python bench.py --variant implicit --no-cpu-baseline > gpurun_out/v_bench_impl.json 2>&1
S="python scripts/sweep.py"
$S --config 3 --variant stream --n 200000 --T 20 > gpurun_out/v_c3.json
$S --config 3 --variant implicit --n 200000 --T 20 > gpurun_out/v_c3i.json
$S --config 4 --T 50 > gpurun_out/v_c4.json
$S --config 5 --variant implicit --n 8388608 --T 2 --reps 2 > gpurun_out/v_c5.json
$S --config 1 --variant stream --T 200 > gpurun_out/v_c1.json
$S --config 1 --variant implicit --T 200 > gpurun_out/v_c1i.json
cat gpurun_out/v_*.json
