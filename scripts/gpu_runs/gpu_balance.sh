# balanced team split + partial-tile skipping: parity then timings
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit or config or stab" 2>&1 | tail -3
S="python scripts/sweep.py"
for c in 1 2; do echo "c$c"; timeout 120 $S --config $c --variant implicit --T 200; done
echo "c5 n=2^20"; timeout 120 $S --config 5 --variant implicit --n 1048576 --T 4
echo "c3"; timeout 300 $S --config 3 --variant implicit --T 20
LSK_TRACE=/tmp/tr_i.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null
python scripts/trace_analyze.py /tmp/tr_i.bin
