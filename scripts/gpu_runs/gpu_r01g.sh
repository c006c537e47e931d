# round-1 (session f) evidence after the boundary work: GPU tests, bench lines, launch list,
# full ncu captures (text summaries + the SASS stall export of the implicit kernel)
set -x
timeout 900 python -m pytest tests -q -m gpu > gpurun_out/r01g_pytest_gpu.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01g_smoke.log 2>&1
python bench.py > gpurun_out/r01g_bench.json 2> gpurun_out/r01g_bench.err
python bench.py --config 5 --steps 3 --warmup 3 --no-alt --no-cpu-baseline --no-e2e > gpurun_out/r01g_bench_config5.json 2>&1
python bench.py --config 4 --steps 3 --warmup 3 --no-alt --no-cpu-baseline --no-e2e > gpurun_out/r01g_bench_config4.json 2>&1
python bench.py --impl reference > gpurun_out/r01g_bench_reference.json 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01g_launches_config2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alt > /dev/null 2>&1
prof() {
  local name=$1; local regex=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$regex -s 1 -c 1 -o /tmp/$name -f "$@" > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 30 > gpurun_out/r01g_${name}_full.txt 2>&1
  python scripts/ncu_lines.py /tmp/$name.ncu-rep 30 > gpurun_out/r01g_${name}_lines.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass > /tmp/${name}_sass.csv 2>/dev/null
  python scripts/sass_stalls.py /tmp/${name}_sass.csv > gpurun_out/r01g_${name}_sass.txt 2>&1
}
prof implicit_c2 implicit_kernel python scripts/prof_one.py --config 2 --variant implicit --T 20

ls -la gpurun_out/ | grep r01g
