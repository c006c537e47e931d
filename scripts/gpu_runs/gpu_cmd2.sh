set -x
python bench.py --variant stream --no-cpu-baseline > gpurun_out/b_stream.json 2> gpurun_out/b_stream.err
python bench.py --variant implicit > gpurun_out/b_impl.json 2> gpurun_out/b_impl.err
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m slow > gpurun_out/slow.log 2>&1
python scripts/prof_one.py --variant stream --T 50 > gpurun_out/p1.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn -s 1 -c 1 -o gpurun_out/prof_stream python scripts/prof_one.py --variant stream --T 50 > gpurun_out/ncu1.log 2>&1
python scripts/prof_one.py --variant implicit --T 50 > gpurun_out/p2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn -s 1 -c 1 -o gpurun_out/prof_impl python scripts/prof_one.py --variant implicit --T 50 > gpurun_out/ncu2.log 2>&1
tail -3 gpurun_out/*.log; cat gpurun_out/b_*.json gpurun_out/b_*.err
