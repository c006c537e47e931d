prof() {
  local name=$1; local regex=$2; shift 2
  ncu --set full --clock-control none --import-source on -k regex:$regex -s 1 -c 1 -o /tmp/$name -f "$@" > /dev/null 2>&1
  python scripts/ncu_summary.py /tmp/$name.ncu-rep 40 > gpurun_out/${name}_full.txt 2>&1
  python scripts/ncu_lines.py /tmp/$name.ncu-rep 40 > gpurun_out/${name}_lines.txt 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/${name}_raw.csv 2>/dev/null
}
prof r01d_implicit_c2 implicit_kernel python scripts/prof_one.py --config 2 --variant implicit --T 20
prof r01d_implicit_c5 implicit_kernel python scripts/prof_one.py --config 5 --n 1048576 --variant implicit --T 2
