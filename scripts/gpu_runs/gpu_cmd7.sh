timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -4
S="python scripts/sweep.py"
$S --variant stream
LSK_GPP=74 $S --variant stream
$S --variant implicit
$S --config 3 --variant stream --n 50000 --T 50
$S --config 1 --variant stream
$S --config 1 --variant implicit
