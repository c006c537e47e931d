timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "implicit or divergence or nccl or smoke" 2>&1 | tail -3
S="python scripts/sweep.py"
$S --variant implicit
LSK_ITEAM=2 $S --variant implicit
LSK_TRACE=gpurun_out/tr_impl4.bin $S --variant implicit --T 30 --reps 1 > /dev/null; python scripts/trace_analyze.py gpurun_out/tr_impl4.bin
$S --config 5 --variant implicit --n 2000000 --T 5
