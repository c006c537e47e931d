timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
S="python scripts/sweep.py --config 4 --T 50"
$S
LSK_BGPP=1 $S
LSK_BGPP=8 $S
