S="python scripts/sweep.py"
LSK_DEBUG=1 $S --variant stream
LSK_DEBUG=1 LSK_NSTAGE=3 $S --variant stream
LSK_DEBUG=1 LSK_GPP=74 $S --variant stream
LSK_DEBUG=1 $S --variant stream --config 3 --n 50000 --T 50
$S --variant stream
python scripts/prof_one.py --variant stream --T 20 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn -s 1 -c 1 -o gpurun_out/prof_stream2 python scripts/prof_one.py --variant stream --T 20 > gpurun_out/ncu3.log 2>&1; tail -2 gpurun_out/ncu3.log
