timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit or config" 2>&1 | tail -3
S="python scripts/sweep.py"
for C in "128,4,2,4,0" "128,2,2,8,1"; do echo "c2 team ICFG=$C"; LSK_IWARP=0 LSK_ICFG=$C timeout 120 $S --config 2 --variant implicit --T 100; done
echo "c5 team default"; timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2
LSK_IWARP=0 LSK_TRACE=/tmp/tr_t.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr_t.bin
