timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "config5" 2>&1 | tail -2
S="python scripts/sweep.py --config 5 --variant implicit --n 2000000 --T 5"
$S
LSK_ITR=2 $S
