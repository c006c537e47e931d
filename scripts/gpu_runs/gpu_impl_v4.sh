# implicit v4: parity + config sweep
timeout 900 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -4
S="python scripts/sweep.py"
for F in 1 0; do
 for C in "" "128,3,2,4" "128,4,2,2" "512,1,2,2" "128,2,2,8"; do
  echo "c2 FACT=$F ICFG=$C"; LSK_FACT=$F LSK_ICFG=$C timeout 120 $S --config 2 --variant implicit --T 100
 done
done
for C in "" "512,1,2,2"; do
 for F in 1 0; do
  echo "c5 FACT=$F ICFG=$C"; LSK_FACT=$F LSK_ICFG=$C timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2
 done
done
echo c1; timeout 60 $S --config 1 --variant implicit --T 200
