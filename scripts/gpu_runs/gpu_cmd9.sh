S="python scripts/sweep.py"
for g in 8 32 74 148; do LSK_DEBUG=1 LSK_GPP=$g $S --variant stream --n 4736 --T 500; done
for g in 148; do LSK_GPP=$g $S --variant stream --n 4736 --T 500; done
