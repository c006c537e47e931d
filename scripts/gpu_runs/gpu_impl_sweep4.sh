S="python scripts/sweep.py"
for C in "128,2,2,16,0" "64,4,4,8,0" "64,4,4,4,0" "64,3,4,8,0"; do echo "c2 $C"; LSK_ICFG=$C timeout 120 $S --config 2 --variant implicit --T 100; done
for C in "128,2,2,16,0"; do echo "c2-5 $C"; LSK_ICFG=$C timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2; done
