timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
S="python scripts/sweep.py"
$S --variant implicit
$S --variant implicit --cps 1
$S --variant implicit --n 4736 --T 500
$S --config 5 --variant implicit --n 2000000 --T 5
