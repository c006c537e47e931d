timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "implicit" 2>&1 | tail -2
python scripts/sweep.py --variant implicit
