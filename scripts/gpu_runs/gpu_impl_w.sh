timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit or config" 2>&1 | tail -3
S="python scripts/sweep.py"
for C in "" "8,8,2"; do
  for F in 1 0; do echo "c2 warp FACT=$F IWCFG=$C"; LSK_FACT=$F LSK_IWCFG=$C timeout 120 $S --config 2 --variant implicit --T 100; done
done
echo "c1 warp"; timeout 60 $S --config 1 --variant implicit --T 200
echo "c1 warp 8,4,4"; LSK_IWCFG=8,4,4 timeout 60 $S --config 1 --variant implicit --T 200
LSK_TRACE=/tmp/tr_w.bin $S --config 2 --variant implicit --T 50 --reps 1 > /dev/null; python scripts/trace_analyze.py /tmp/tr_w.bin
