timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit or config or stab or tol" 2>&1 | tail -2
AB_C5=1 AB_C1=1 bash scripts/gpu_runs/gpu_ab.sh main prev
LSK_TRACE=/tmp/tr.bin timeout 120 python scripts/sweep.py --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr.bin
