# round-1 (session c) evidence: bench line, launch list of the same bench command, full ncu
# captures of the dominant kernels (text summaries only)
set -x
python bench.py > gpurun_out/r01c_bench.json 2> gpurun_out/r01c_bench.err
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/r01c_launches_config2.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-alt > /dev/null 2>&1
prof() {
  local name=$1; local regex=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$regex -s 1 -c 1 -o /tmp/$name -f "$@" > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 30 > gpurun_out/r01c_${name}_full.txt 2>&1
  python scripts/ncu_lines.py /tmp/$name.ncu-rep 30 > gpurun_out/r01c_${name}_lines.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > /tmp/${name}_raw.csv 2>/dev/null
  python - "$name" <<'PY'
import csv, sys
rows = list(csv.reader(open('/tmp/%s_raw.csv' % sys.argv[1])))
h, u, v = rows[0], rows[1], rows[2]
keep = [k for k in h if k.startswith('smsp__average_warps_issue_stalled_') and k.endswith('_per_issue_active.ratio')]
out = sorted(((float(v[h.index(k)]), k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')) for k in keep), reverse=True)[:8]
with open('gpurun_out/r01c_%s_full.txt' % sys.argv[1], 'a') as f:
    f.write('\nwarp stall reasons (per issued instruction):\n')
    for val, k in out: f.write('  %-24s %.3f\n' % (k, val))
PY
}
prof implicit_c2 implicit_kernel python scripts/prof_one.py --config 2 --variant implicit --T 20
prof implicit_c5 implicit_kernel python scripts/prof_one.py --config 5 --n 1048576 --variant implicit --T 2
prof stream_c2 sinkhorn_kernel python scripts/prof_one.py --config 2 --variant stream --T 20
prof accel_pass_c2 pass_kernel python scripts/sweep.py --config 2 --variant accel --T 3 --reps 1
ls -la gpurun_out/ | grep r01c
