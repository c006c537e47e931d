S="python scripts/sweep.py"
for G in 0 1 2 4 8; do for V in implicit stream; do echo "c1 gpp=$G $V"; LSK_GPP=$G $S --config 1 --variant $V --T 200 | sed 's/"env".*"cps": 0, //'; done; done
for G in 0 1 2; do echo "c2-small(4000) gpp=$G"; LSK_GPP=$G $S --config 2 --n 4000 --variant implicit --T 100 | sed 's/"env".*"cps": 0, //'; done
