# official bench line + reference arm + ncu launch list + one full capture (round-1 evidence)
python bench.py > gpurun_out/bench_r1.json 2> gpurun_out/bench_r1.err
python bench.py --impl reference > gpurun_out/bench_ref_r1.json 2> gpurun_out/bench_ref_r1.err
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv $CMD > gpurun_out/ncu_launch.log 2>&1
$CMD > gpurun_out/plain2.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:sinkhorn -s 3 -c 1 -o gpurun_out/prof_bench_r1 $CMD > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/bench_r1.json gpurun_out/bench_ref_r1.json; tail -n 2 gpurun_out/ncu_full.log
