timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "implicit or config" 2>&1 | tail -3
S="python scripts/sweep.py"
for C in "" "128,2,2,8,1" "128,2,2,4,1" "256,1,2,4,1"; do
  for F in 1 0; do echo "c2 FACT=$F ICFG=$C"; LSK_FACT=$F LSK_ICFG=$C timeout 120 $S --config 2 --variant implicit --T 100; done
done
for C in "" "256,1,4,2,1"; do
  for F in 1 0; do echo "c5 FACT=$F ICFG=$C"; LSK_FACT=$F LSK_ICFG=$C timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2; done
done
