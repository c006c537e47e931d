S="python scripts/sweep.py"
LSK_DEBUG=1 $S --variant stream --n 4736 --T 500
$S --variant stream --n 4736 --T 500
$S --variant stream
LSK_TR=16 $S --variant stream
LSK_TR=32 $S --variant stream
LSK_DEBUG=1 $S --variant stream
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
