#!/bin/bash
# round 2 (session 4): GPU suite, bench line, launch list and implicit capture after the boundary round-trip trims
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -q -m gpu > $O/s21_pytest_gpu.log 2>&1
echo "suite rc=$?" >> $O/s21_pytest_gpu.log
tail -n 4 $O/s21_pytest_gpu.log
timeout 900 python bench.py > $O/s21_bench.json 2> $O/s21_bench.err
echo "bench rc=$?" >> $O/s21_bench.err
tail -n 2 $O/s21_bench.err
CMD="python bench.py --steps 2 --warmup 3 --no-extra --no-e2e --no-cpu-baseline --no-alt"
timeout 300 $CMD > $O/s21_plain.json 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/s21_launches.csv $CMD > $O/s21_ncu_launches.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:implicit_kernel -s 3 -c 1 -o $O/s21_implicit -f $CMD > $O/s21_ncu_full.log 2>&1
python scripts/ncu_summary.py $O/s21_implicit.ncu-rep 30 > $O/s21_implicit_c2_summary.txt 2>&1
rm -f $O/*.ncu-rep
python - <<'PY'
import json
d=json.load(open("gpurun_out/s21_bench.json"))
print("headline", d["value"], d["roofline"]["frac"], d["e2e"]["value"] if d.get("e2e") else None, d["clocks"])
for k,v in d.get("configs",{}).items(): print(k, v["value"], v["roofline"]["bound"], v["roofline"]["frac"], v["config"].get("variant"), v.get("clocks"))
for a in d.get("alt_variants",[]): print("alt", a["variant"], a["value"], a["roofline"]["frac"])
PY
head -12 $O/s21_implicit_c2_summary.txt
