S="python scripts/sweep.py"
for V in stream implicit; do echo "c2 $V"; timeout 120 $S --config 2 --variant $V --T 100; done
echo c3; timeout 120 $S --config 3 --variant stream --n 200000 --T 20
echo c5; timeout 120 $S --config 5 --variant implicit --n 1048576 --T 2
