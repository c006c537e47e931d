prof() {  # name, then the command
  local name=$1; shift
  ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 1 -c 1 \
    -o /tmp/$name -f "$@" > gpurun_out/ncu_$name.log 2>&1
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 30 > gpurun_out/sum_$name.txt 2>&1
  python scripts/ncu_lines.py /tmp/$name.ncu-rep 40 > gpurun_out/lines_$name.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/raw_$name.csv 2>/dev/null
}
LSK_ICFG=128,2,2,8 prof impl4_c2 python scripts/prof_one.py --config 2 --variant implicit --T 20
prof impl4_c5 python scripts/prof_one.py --config 5 --n 1048576 --variant implicit --T 2
