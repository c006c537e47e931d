timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
S="python scripts/sweep.py"
$S --variant stream
LSK_DEBUG=1 $S --variant stream
$S --config 3 --variant stream --n 100000 --T 50
$S --config 3 --variant stream --n 200000 --T 20
LSK_DEBUG=1 $S --config 3 --variant stream --n 200000 --T 20
$S --config 4 --T 50
$S --config 4 --T 50 --cps 1
$S --config 5 --variant stream --n 2000000 --T 5
$S --config 5 --variant implicit --n 2000000 --T 5
$S --variant implicit
