timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "implicit or divergence or nccl or smoke" 2>&1 | tail -2
python scripts/sweep.py --variant implicit
LSK_ITEAM=2 python scripts/sweep.py --variant implicit
python scripts/sweep.py --config 5 --variant implicit --n 2000000 --T 5
