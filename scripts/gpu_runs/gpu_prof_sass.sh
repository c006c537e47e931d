# full capture of the config-2 implicit kernel (short solve) for SASS-level stall analysis
python scripts/sweep.py --config 2 --variant implicit --T 20 --reps 1 > /dev/null
ncu --set full --import-source on --clock-control none -k regex:implicit_kernel -c 1 -o gpurun_out/ic2 \
  python scripts/sweep.py --config 2 --variant implicit --T 20 --reps 1 > gpurun_out/ic2.log 2>&1
ncu -i gpurun_out/ic2.ncu-rep --page source --csv --print-source sass > gpurun_out/ic2_sass.csv 2> gpurun_out/ic2_sass.err
ls -la gpurun_out/ic2*
