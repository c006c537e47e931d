# ncu full capture of the implicit kernel, config 2 (T=20) and config 5 reduced (n=1M, T=2)
python scripts/prof_one.py --config 2 --variant implicit --T 20 > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 1 -c 1 \
  -o gpurun_out/impl_c2 -f python scripts/prof_one.py --config 2 --variant implicit --T 20 > gpurun_out/ncu_impl_c2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 1 -c 1 \
  -o gpurun_out/impl_c5 -f python scripts/prof_one.py --config 5 --n 1048576 --variant implicit --T 2 > gpurun_out/ncu_impl_c5.log 2>&1
ls -la gpurun_out/
