timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -8
S="python scripts/sweep.py"
$S --variant stream
for g in 74; do LSK_GPP=$g $S --variant stream; done
LSK_NSTAGE=3 $S --variant stream
$S --variant stream --n 1184
$S --variant implicit
$S --variant implicit --n 1184
$S --config 3 --variant stream --n 50000 --T 50
$S --config 5 --variant implicit --n 1000000 --T 5
