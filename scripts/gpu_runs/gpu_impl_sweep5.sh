S="python scripts/sweep.py"
for C in "512,1,2,4,0" "256,1,4,4,0" "256,1,4,8,0"; do echo "c5 $C"; LSK_ICFG=$C timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2; done
