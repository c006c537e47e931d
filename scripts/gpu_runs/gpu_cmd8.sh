python scripts/prof_one.py --variant implicit --T 20 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn -s 1 -c 1 -o gpurun_out/prof_impl3 python scripts/prof_one.py --variant implicit --T 20 > gpurun_out/ncu4.log 2>&1
python scripts/prof_one.py --variant stream --T 20 > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn -s 1 -c 1 -o gpurun_out/prof_stream3 python scripts/prof_one.py --variant stream --T 20 > gpurun_out/ncu5.log 2>&1
tail -1 gpurun_out/ncu4.log gpurun_out/ncu5.log
