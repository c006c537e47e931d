S="python scripts/sweep.py"
$S --variant stream
for g in 16 37 74 111; do LSK_GPP=$g $S --variant stream; done
for ns in 2 3 4; do LSK_NSTAGE=$ns $S --variant stream; done
$S --variant stream --n 1184
$S --variant stream --n 148
$S --variant stream --n 14800
$S --variant implicit
for g in 37 74; do LSK_GPP=$g $S --variant implicit; done
$S --variant implicit --n 1184
