S="python scripts/sweep.py"
for C in "128,4,2,4,0" "128,3,2,8,0" "128,3,2,4,0" "256,2,1,8,0" "128,4,2,8,0"; do echo "c2 $C"; LSK_ICFG=$C timeout 120 $S --config 2 --variant implicit --T 100; done
for C in "512,1,2,4,0" "384,1,3,4,0" "384,1,3,2,0" "256,2,2,4,0"; do echo "c5 $C"; LSK_ICFG=$C timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2; done
