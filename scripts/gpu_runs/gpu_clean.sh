timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -3
S="python scripts/sweep.py"
$S --config 2 --variant stream --T 100
$S --config 3 --variant stream --n 200000 --T 20
$S --config 4 --T 50
