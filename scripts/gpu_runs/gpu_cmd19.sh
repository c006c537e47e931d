timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "feature_map and 4" 2>&1 | tail -15
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "config4" 2>&1 | tail -5
timeout 300 python scripts/sweep.py --config 4 --T 50 --cps 1
LSK_FEATURE_FFMA=1 timeout 300 python scripts/sweep.py --config 4 --T 5 --cps 1
